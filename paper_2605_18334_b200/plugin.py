"""Blend-kernel plugin with the reference's operator interface.

The reference selects its blend kernels through raster/backend.py:41-43: a
module exposing ``forward_tiles`` and ``backward_tiles`` with the signatures
of raster/_core.pyx:169-170 / :315-317 (numpy in, numpy out, fp64 / int64).
This module provides exactly that interface on top of the sm_100a kernels
(ssg_blend_forward / ssg_blend_backward_slots in libssg_b200.so), so a
reference checkout can register it as a third backend:

    forward_tiles(mean2d, conic, skew2d, opair, color, inst_prim, ranges,
                  tiles_x, width, height, background)
        -> (img (H,W,3) f64, final_T (H,W) f64, n_contrib (H,W) i32,
            last_idx (H,W) i64)
    backward_tiles(..., final_T, last_idx, dL_dpix) -> slots (M,12) f64

Screen quantities are handed over in fp64 and rounded to the kernels' fp32
(the mean stays fp64 so blend offsets are formed exactly).  There is no CPU
fallback: a missing or failing extension raises.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as N

CORE_BUILD = 1
KERNELS = 1

_SPLAT = np.dtype([("mean", "<f8", 2), ("conic", "<f4", 3), ("skew", "<f4", 2), ("opair", "<f4", 2),
                   ("rgb", "<f4", 3), ("pad", "<u4", 2)])
assert _SPLAT.itemsize == N.SPLAT_BYTES


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _splats(mean2d, conic, skew2d, opair, color) -> torch.Tensor:
    n = np.asarray(mean2d).shape[0]
    rec = np.zeros(n, dtype=_SPLAT)
    rec["mean"] = np.asarray(mean2d, dtype=np.float64).reshape(n, 2)
    rec["conic"] = np.asarray(conic, dtype=np.float64).reshape(n, 3)
    rec["skew"] = np.asarray(skew2d, dtype=np.float64).reshape(n, 2)
    rec["opair"] = np.asarray(opair, dtype=np.float64).reshape(n, 2)
    rec["rgb"] = np.asarray(color, dtype=np.float64).reshape(n, 3)
    return torch.from_numpy(rec.view(np.uint8)).to(_device())


def _bins(inst_prim, ranges):
    dev = _device()
    ip = torch.from_numpy(np.ascontiguousarray(inst_prim, dtype=np.int64).astype(np.int32)).to(dev)
    rg = torch.from_numpy(np.ascontiguousarray(ranges, dtype=np.int64).astype(np.int32)).to(dev)
    b = N.SsgBinBuffers()
    b.capacity = int(ip.numel())
    b.inst_prim = ip.data_ptr() if ip.numel() else None
    b.ranges = rg.data_ptr()
    return b, (ip, rg)


def _check_dims(width, height, ranges, tiles_x):
    if width > 65535 or height > 65535:
        raise ValueError("image dimension overflow")
    if tiles_x != -(-width // 16) or np.asarray(ranges).shape[0] != tiles_x * -(-height // 16):
        raise ValueError("ranges / tiles_x do not match the image size")


def forward_tiles(mean2d, conic, skew2d, opair, color, inst_prim, ranges, tiles_x, width, height,
                  background):
    """raster/_core.pyx:169-200 on the GPU."""
    _check_dims(width, height, ranges, tiles_x)
    L = N.lib()
    dev = _device()
    sp = _splats(mean2d, conic, skew2d, opair, color)
    b, keep = _bins(inst_prim, ranges)
    color_d = torch.empty((height, width, 3), dtype=torch.float32, device=dev)
    T_d = torch.empty((height, width), dtype=torch.float32, device=dev)
    nc_d = torch.empty((height, width), dtype=torch.int32, device=dev)
    li_d = torch.empty((height, width), dtype=torch.int32, device=dev)
    f = N.SsgFrameBuffers()
    f.color, f.final_T, f.n_contrib, f.last_idx = (color_d.data_ptr(), T_d.data_ptr(), nc_d.data_ptr(),
                                                   li_d.data_ptr())
    bg = (ctypes.c_float * 3)(*[float(x) for x in np.asarray(background, dtype=np.float64).reshape(3)])
    N.check(L.ssg_blend_forward(b.capacity, width, height, bg, sp.data_ptr() if sp.numel() else None,
                                ctypes.byref(b), ctypes.byref(f), torch.cuda.current_stream().cuda_stream),
            "ssg_blend_forward")
    out = (color_d.double().cpu().numpy(), T_d.double().cpu().numpy(), nc_d.cpu().numpy(),
           li_d.long().cpu().numpy())
    del keep
    return out


def backward_tiles(mean2d, conic, skew2d, opair, color, inst_prim, ranges, tiles_x, width, height,
                   background, final_T, last_idx, dL_dpix):
    """raster/_core.pyx:315-343 on the GPU: per-instance slots (M,12)."""
    _check_dims(width, height, ranges, tiles_x)
    L = N.lib()
    dev = _device()
    sp = _splats(mean2d, conic, skew2d, opair, color)
    b, keep = _bins(inst_prim, ranges)
    m = b.capacity
    T_d = torch.from_numpy(np.ascontiguousarray(final_T, dtype=np.float64)).to(dev).float()
    li_d = torch.from_numpy(np.ascontiguousarray(last_idx, dtype=np.int64)).to(dev).int()
    dL_d = torch.from_numpy(np.ascontiguousarray(dL_dpix, dtype=np.float64)).to(dev).float()
    slots = torch.empty((max(m, 1), 12), dtype=torch.float32, device=dev)
    f = N.SsgFrameBuffers()
    f.final_T, f.last_idx = T_d.data_ptr(), li_d.data_ptr()
    bg = (ctypes.c_float * 3)(*[float(x) for x in np.asarray(background, dtype=np.float64).reshape(3)])
    N.check(L.ssg_blend_backward_slots(m, width, height, bg, sp.data_ptr() if sp.numel() else None,
                                       ctypes.byref(b), ctypes.byref(f), dL_d.data_ptr(), slots.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream),
            "ssg_blend_backward_slots")
    out = slots[:m].double().cpu().numpy()
    del keep
    return out
