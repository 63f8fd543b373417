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

def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _splats(mean2d, conic, skew2d, opair, color):
    """Device screen records (fp32 splat with its alpha band + the fp64 twin
    the threshold-band path reads) built by ssg_pack_splats from the fp64
    plugin inputs."""
    n = int(np.asarray(mean2d).shape[0])
    dev = _device()

    def up(a, w):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(n, w)).to(dev)

    ins = [up(mean2d, 2), up(conic, 3), up(skew2d, 2), up(opair, 2), up(color, 3)]
    sp = torch.empty((max(n, 1), N.SPLAT_BYTES // 8), dtype=torch.float64, device=dev)
    sp64 = torch.empty((max(n, 1), N.SPLAT64_BYTES // 8), dtype=torch.float64, device=dev)
    N.check(N.lib().ssg_pack_splats(n, *[t.data_ptr() for t in ins], sp.data_ptr(), sp64.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream), "ssg_pack_splats")
    return sp, sp64


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
    sp, sp64 = _splats(mean2d, conic, skew2d, opair, color)
    b, keep = _bins(inst_prim, ranges)
    ntx, nty = tiles_x, -(-height // 16)
    redo, rlist, rcount, _ = _decision_buffers(0, ntx, nty, width, height, dev)
    color_d = torch.empty((height, width, 3), dtype=torch.float32, device=dev)
    T_d = torch.empty((height, width), dtype=torch.float32, device=dev)
    nc_d = torch.empty((height, width), dtype=torch.int32, device=dev)
    li_d = torch.empty((height, width), dtype=torch.int32, device=dev)
    f = N.SsgFrameBuffers()
    f.color, f.final_T, f.n_contrib, f.last_idx = (color_d.data_ptr(), T_d.data_ptr(), nc_d.data_ptr(),
                                                   li_d.data_ptr())
    f.redo_mask, f.redo_list, f.redo_count = redo.data_ptr(), rlist.data_ptr(), rcount.data_ptr()
    bg = (ctypes.c_float * 3)(*[float(x) for x in np.asarray(background, dtype=np.float64).reshape(3)])
    N.check(L.ssg_blend_forward(b.capacity, width, height, bg, sp.data_ptr(), sp64.data_ptr(),
                                ctypes.byref(b), ctypes.byref(f), torch.cuda.current_stream().cuda_stream),
            "ssg_blend_forward")
    out = (color_d.double().cpu().numpy(), T_d.double().cpu().numpy(), nc_d.cpu().numpy(),
           li_d.long().cpu().numpy())
    del keep
    return out


def _decision_buffers(m, ntx, nty, width, height, dev):
    redo = torch.empty((max(ntx * nty, 1) * 8,), dtype=torch.int32, device=dev)
    rlist = torch.empty((max(width * height, 1),), dtype=torch.int32, device=dev)
    rcount = torch.empty((1,), dtype=torch.int32, device=dev)
    words = int(N.lib().ssg_blend_mask_words(max(m, 1), max(ntx * nty, 1)))
    bmask = torch.empty((max(words, 1),), dtype=torch.int32, device=dev)
    return redo, rlist, rcount, bmask


def backward_tiles(mean2d, conic, skew2d, opair, color, inst_prim, ranges, tiles_x, width, height,
                   background, final_T, last_idx, dL_dpix):
    """raster/_core.pyx:315-343 on the GPU: per-instance slots (M,12),
    deterministic (fixed-order combination, no atomics).  The decision
    records the backward needs (blend mask, exact-path pixels) come from a
    forward pass over the same inputs; its decisions are the reference's,
    so they agree with the caller's final_T / last_idx."""
    _check_dims(width, height, ranges, tiles_x)
    L = N.lib()
    dev = _device()
    sp, sp64 = _splats(mean2d, conic, skew2d, opair, color)
    b, keep = _bins(inst_prim, ranges)
    m = b.capacity
    ntx, nty = tiles_x, -(-height // 16)
    T_d = torch.from_numpy(np.ascontiguousarray(final_T, dtype=np.float64)).to(dev).float()
    li_d = torch.from_numpy(np.ascontiguousarray(last_idx, dtype=np.int64)).to(dev).int()
    dL_d = torch.from_numpy(np.ascontiguousarray(dL_dpix, dtype=np.float64)).to(dev).float()
    slots = torch.empty((max(m, 1), 12), dtype=torch.float32, device=dev)
    redo, rlist, rcount, bmask = _decision_buffers(m, ntx, nty, width, height, dev)
    scratch = [torch.empty((height, width, 3), dtype=torch.float32, device=dev),
               torch.empty((height, width), dtype=torch.float32, device=dev),
               torch.empty((height, width), dtype=torch.int32, device=dev),
               torch.empty((height, width), dtype=torch.int32, device=dev)]
    bg = (ctypes.c_float * 3)(*[float(x) for x in np.asarray(background, dtype=np.float64).reshape(3)])
    st = torch.cuda.current_stream().cuda_stream
    fw = N.SsgFrameBuffers()
    fw.color, fw.final_T, fw.n_contrib, fw.last_idx = (t.data_ptr() for t in scratch)
    fw.blend_mask, fw.redo_mask, fw.redo_list, fw.redo_count = (bmask.data_ptr(), redo.data_ptr(), rlist.data_ptr(),
                                                                rcount.data_ptr())
    N.check(L.ssg_blend_forward(m, width, height, bg, sp.data_ptr(), sp64.data_ptr(), ctypes.byref(b),
                                ctypes.byref(fw), st), "ssg_blend_forward (decision records)")
    f = N.SsgFrameBuffers()
    f.final_T, f.last_idx = T_d.data_ptr(), li_d.data_ptr()
    f.blend_mask, f.redo_mask, f.redo_list, f.redo_count = (bmask.data_ptr(), redo.data_ptr(), rlist.data_ptr(),
                                                            rcount.data_ptr())
    N.check(L.ssg_blend_backward_slots(m, width, height, bg, sp.data_ptr(), sp64.data_ptr(),
                                       ctypes.byref(b), ctypes.byref(f), dL_d.data_ptr(), slots.data_ptr(), st),
            "ssg_blend_backward_slots")
    out = slots[:m].double().cpu().numpy()
    del keep
    return out


def set_num_threads(n: int) -> None:
    """raster/_core.pyx:38-39.  The GPU kernels have no host thread pool; the
    call is accepted (and validated) so reference callers keep working."""
    if int(n) < 1:
        raise ValueError("number of threads must be >= 1")


def get_max_threads() -> int:
    """raster/_core.pyx:42-43: the parallel width of the blend, i.e. the
    device's resident threads (SMs x max threads per SM)."""
    p = torch.cuda.get_device_properties(_device())
    return int(p.multi_processor_count * p.max_threads_per_multi_processor)


def erf_probe(x):
    """raster/_core.pyx:46-54: the compiled erf evaluated on an array, here
    the fp64 c_erf restatement the blend kernels' threshold path runs on the
    device (ssg_erf_probe); same shape as x."""
    xv = np.ascontiguousarray(x, dtype=np.float64)
    flat = torch.from_numpy(xv.ravel()).to(_device())
    out = torch.empty_like(flat)
    N.check(N.lib().ssg_erf_probe(flat.data_ptr() if flat.numel() else None, int(flat.numel()), None,
                                  out.data_ptr() if flat.numel() else None,
                                  torch.cuda.current_stream().cuda_stream), "ssg_erf_probe")
    return out.cpu().numpy().reshape(np.shape(x))


def erf_probe_fp32(x):
    """E - 1 of the fp32 blend path (1 + erf(z) evaluated as erfc(-z) with the
    kernels' fast erfc), for accuracy checks against the reference erf."""
    xv = np.ascontiguousarray(x, dtype=np.float64)
    flat = torch.from_numpy(xv.ravel()).to(_device())
    out = torch.empty(flat.shape, dtype=torch.float32, device=flat.device)
    N.check(N.lib().ssg_erf_probe(flat.data_ptr() if flat.numel() else None, int(flat.numel()),
                                  out.data_ptr() if flat.numel() else None, None,
                                  torch.cuda.current_stream().cuda_stream), "ssg_erf_probe")
    return out.double().cpu().numpy().reshape(np.shape(x)) - 1.0
