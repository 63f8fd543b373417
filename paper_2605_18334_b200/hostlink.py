"""Host <-> device copies of caller arrays.

Pageable host arrays (what a reference caller passes) cross the link at ~11
GB/s when the driver stages them itself; a multi-threaded host copy into
page-locked memory runs at ~45 GB/s on the GPU hosts and the pinned copy to
the device at ~55 GB/s (tools/memcpy_probe.py).  So pageable sources go
through two pinned staging buffers in turns: the host fills one while the
other is on the link.  Pinned sources copy asynchronously as they are."""

from __future__ import annotations

import threading

import numpy as np
import torch

STAGE_BYTES = 64 << 20
_STAGING: dict = {}
_STAGING_LOCK = threading.Lock()


def is_pinned(a: np.ndarray) -> bool:
    return bool(torch.from_numpy(a).is_pinned()) if a.size else True


def _stage_ring(dev):
    key = str(dev)
    with _STAGING_LOCK:
        if key not in _STAGING:
            _STAGING[key] = {"slots": [[torch.empty(STAGE_BYTES, dtype=torch.uint8, pin_memory=True), None]
                                       for _ in range(2)], "next": 0, "lock": threading.Lock()}
        return _STAGING[key]


def to_device(a: np.ndarray, dev, pinned: bool | None = None) -> torch.Tensor:
    """A C-contiguous host array on the device (same dtype), queued on the
    current stream.  Pinned arrays copy asynchronously; pageable ones are
    staged (the call returns once the last piece is in staging, the copies
    to the device still queued)."""
    if pinned is None:
        pinned = is_pinned(a)
    src = torch.from_numpy(a)
    if pinned:
        return src.to(dev, non_blocking=True)
    out = torch.empty(src.shape, dtype=src.dtype, device=dev)
    flat_src, flat_out = src.reshape(-1), out.reshape(-1)
    per = max(STAGE_BYTES // src.element_size(), 1)
    ring = _stage_ring(dev)
    st = torch.cuda.current_stream(dev)
    with ring["lock"]:
        for lo in range(0, flat_src.numel(), per):
            hi = min(lo + per, flat_src.numel())
            slot = ring["slots"][ring["next"]]
            ring["next"] ^= 1
            if slot[1] is not None:
                slot[1].synchronize()  # its previous piece has left the buffer
            buf = slot[0][:(hi - lo) * src.element_size()].view(src.dtype)
            buf.copy_(flat_src[lo:hi])  # multi-threaded host copy
            flat_out[lo:hi].copy_(buf, non_blocking=True)
            slot[1] = torch.cuda.Event()
            slot[1].record(st)
    return out
