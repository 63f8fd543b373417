"""Adaptive density control on the device.

densify_and_prune mirrors optimize/densify.py:24-116 on a DeviceScene: tau_z
calibration (90th percentile of g_z when NaN, written back into cfg like the
reference), clone / split / prune flags, the new primitive set in the
reference's row order ([kept | clones | split children]), the Adam moment
remap (adam.py:99-110), the non-finite check (FloatingPointError) and the
in-place zeroing of the depth-gradient statistic.  Two native calls:
ssg_densify_plan (flags, counts; one synchronisation for the new size) and
ssg_densify_apply (every output row written once).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _native as N
from .engine import DeviceScene


def _ptr(t):
    return None if t is None else t.data_ptr()


def densify_and_prune(ds: DeviceScene, stats, cfg, adam=None, max_radii=None) -> dict:
    """stats: g_uv (n) fp64, g_z (n) fp32, d_mu (n,3) fp64 device tensors
    (IntervalStats.bundle()); mutates ds, adam, cfg.tau_z and stats.g_z."""
    tr = getattr(adam, "_trainer", None)
    if tr is not None and getattr(tr, "pipelined", False):
        tr.flush()  # resolve the last pipelined step before the scene changes
    n = ds.n
    report = {"n_cloned": 0, "n_split": 0, "n_pruned": 0, "n_primitives": n}
    if n == 0:
        return report
    dev = ds.mu.device
    L = N.lib()
    g_uv = stats.g_uv.to(device=dev, dtype=torch.float64).contiguous()
    g_z = stats.g_z.to(device=dev, dtype=torch.float32).contiguous()
    d_mu = stats.d_mu.to(device=dev, dtype=torch.float64).contiguous()
    st = N.SsgDensifyStats(g_uv.data_ptr(), g_z.data_ptr(), d_mu.data_ptr())
    radii = None
    if max_radii is not None and cfg.max_screen_radius is not None:
        radii = torch.as_tensor(np.asarray(max_radii, dtype=np.float64) if not torch.is_tensor(max_radii)
                                else max_radii, dtype=torch.float64, device=dev).contiguous()
    c = N.SsgDensifyCfg(cfg.tau_uv, cfg.tau_z, cfg.split_scale_threshold, cfg.prune_alpha,
                        float(cfg.max_screen_radius) if radii is not None else -1.0,
                        cfg.position_lr_at(cfg.densify_start), _ptr(radii))
    flags = torch.empty(n, dtype=torch.uint8, device=dev)
    temp = torch.empty(int(L.ssg_densify_temp_bytes(n)), dtype=torch.uint8, device=dev)
    counts = (ctypes.c_int64 * 4)()
    tau = ctypes.c_double(0.0)
    stream = torch.cuda.current_stream(dev).cuda_stream
    sc = ds.struct()
    N.check(L.ssg_densify_plan(ctypes.byref(sc), ctypes.byref(st), ctypes.byref(c), flags.data_ptr(),
                               temp.data_ptr(), temp.numel(), counts, ctypes.byref(tau), stream),
            "ssg_densify_plan")
    if math.isnan(cfg.tau_z):
        cfg.tau_z = float(tau.value)  # densify.py:39-40
    n_keep, n_clone, n_split, n_pruned = (int(x) for x in counts)
    n_new = n_keep + n_clone + 2 * n_split
    report.update(n_pruned=n_pruned, n_cloned=n_clone, n_split=n_split)

    K = ds.K
    z64 = lambda *s: torch.empty(s, dtype=torch.float64, device=dev)  # noqa: E731
    z32 = lambda *s: torch.empty(s, dtype=torch.float32, device=dev)  # noqa: E731
    m = max(n_new, 1)
    new = dict(mu=z64(m, 3), log_scale=z64(m, 3), rot=z64(m, 4), sh=z32(m, K, 3), opacity_logits=z32(m, 2),
               beta=z32(m, 3), dir=z32(m, 3))
    p = N.SsgParams()
    p.n, p.sh_degree, p.sh_coeffs = n_new, ds.sh_degree, K
    for f, t in new.items():
        setattr(p, f, t.data_ptr())
    a_in = a_out = None
    if adam is not None:
        new_m = {k: torch.empty((m,) + tuple(v.shape[1:]), dtype=torch.float32, device=dev) for k, v in adam.m.items()}
        new_v = {k: torch.empty_like(v) for k, v in new_m.items()}
        a_in, a_out = N.SsgAdamState(), N.SsgAdamState()
        for f in adam.FIELDS:
            setattr(a_in, "m_" + f, adam.m[f].data_ptr())
            setattr(a_in, "v_" + f, adam.v[f].data_ptr())
            setattr(a_out, "m_" + f, new_m[f].data_ptr())
            setattr(a_out, "v_" + f, new_v[f].data_ptr())
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    N.check(L.ssg_densify_apply(ctypes.byref(sc), ctypes.byref(p),
                                ctypes.byref(a_in) if a_in is not None else None,
                                ctypes.byref(a_out) if a_out is not None else None,
                                ctypes.byref(st), ctypes.byref(c), flags.data_ptr(), temp.data_ptr(),
                                bad.data_ptr(), stream), "ssg_densify_apply")
    # the new set replaces the old one in place (the train loop holds ds)
    for f, t in new.items():
        setattr(ds, f, t[:n_new])
    ds.n = n_new
    if adam is not None:
        adam.m = {k: v[:n_new] for k, v in new_m.items()}
        adam.v = {k: v[:n_new] for k, v in new_v.items()}
        adam.row_ok = torch.empty(max(n_new, 1), dtype=torch.uint8, device=dev)
    report["n_primitives"] = n_new
    if int(bad.item()):
        for f in ("mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir"):
            if not bool(torch.isfinite(getattr(ds, f)).all()):
                raise FloatingPointError(f"densification produced non-finite {f}")  # densify.py:112-114
    stats.g_z.zero_()  # densify.py:115
    return report
