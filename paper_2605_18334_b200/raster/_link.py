"""Host-link helpers of the drop-in calls: the copy streams, the host scene
as fp64 arrays in the device layout, and the on-device bitwise comparison
of two device scenes (the check that makes a speculative result exact)."""

from __future__ import annotations

import contextlib

import numpy as np
import torch

from ..hostlink import is_pinned, to_device  # noqa: F401  (re-exported)

SCENE_FIELDS = ("mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir")
_INT_VIEW = {torch.float64: torch.int64, torch.float32: torch.int32}
_STREAMS: dict = {}


@contextlib.contextmanager
def drain_on_error(dev):
    """Context for a speculative call: if it raises, wait for the copy
    streams before the exception propagates (their transfers target buffers
    the unwinding frees)."""
    try:
        yield
    except BaseException:
        for st in copy_streams(dev):
            st.synchronize()
        raise


def copy_streams(dev) -> tuple:
    """(host->device, device->host) streams of a device, created once."""
    key = str(dev)
    if key not in _STREAMS:
        _STREAMS[key] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return _STREAMS[key]


def host_fields(scene, n: int, K: int) -> dict:
    """The scene's fields as C-contiguous fp64 arrays shaped like the device
    copy (no copy when they already are, e.g. pinned caller arrays)."""
    shapes = {"mu": (n, 3), "log_scale": (n, 3), "rot": (n, 4), "sh": (n, K, 3), "opacity_logits": (n, 2),
              "beta": (n, 3), "dir": (n, 3)}
    out = {}
    for f, shp in shapes.items():
        a = np.asarray(getattr(scene, f))
        if f == "sh":
            a = a.reshape(n, -1, 3)[:, :K, :]
        out[f] = np.ascontiguousarray(a, dtype=np.float64).reshape(shp)
    return out


def host_empty(shape, dtype) -> torch.Tensor:
    """Output buffer of a drop-in call: page-locked (fast, asynchronous
    device->host copies) when the pinned pool can grow, else ordinary host
    memory (the copies then run synchronously, same bytes)."""
    try:
        return torch.empty(shape, dtype=dtype, pin_memory=True)
    except RuntimeError:
        return torch.empty(shape, dtype=dtype)


def upload_rows(ds, srcs: dict, a: int, b: int, dev, pinned: dict | None = None) -> list:
    """Host -> device copies of rows [a, b) of every field, queued on the
    current stream: fp64 fields straight into `ds`, the fields `ds` keeps in
    fp32 as fp64 device temporaries.  Returns the (destination, temporary)
    conversions, which the caller runs on its compute stream once the
    upload's event has passed -- a conversion kernel queued on the copy
    stream would wait there for SM slots behind the compute stream's kernels
    and hold up the copies behind it."""
    conv = []
    for f in SCENE_FIELDS:
        dst, src = getattr(ds, f)[a:b], srcs[f][a:b]
        pin = is_pinned(src) if pinned is None else pinned[f]
        if dst.dtype == torch.float64 and pin:
            dst.copy_(torch.from_numpy(src), non_blocking=True)
        elif dst.dtype == torch.float64:
            dst.copy_(to_device(src, dev, False))  # device-to-device: a copy-engine transfer
        else:
            conv.append((dst, to_device(src, dev, pin)))
    return conv


def finish_rows(conv: list, stream) -> None:
    """Run upload_rows' conversions on `stream` (current stream context)."""
    for dst, tmp in conv:
        dst.copy_(tmp)
        tmp.record_stream(stream)


def scenes_differ(a, b) -> torch.Tensor:
    """Device bool: any bit of any field differs (NaN-safe: compared as
    integers).  No host synchronisation."""
    return torch.stack([(getattr(a, f).view(_INT_VIEW[getattr(a, f).dtype]) !=
                         getattr(b, f).view(_INT_VIEW[getattr(b, f).dtype])).any() for f in SCENE_FIELDS]).any()
