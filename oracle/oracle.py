"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the C oracle (ssg_oracle.c).

The oracle is a CPU fp64 restatement of the reference rasterizer hot path
(pkg/src/skewsplat/raster/{forward,backward,tiles,_core}, projection.py).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; the product package never does.

Functions mirror the reference call chain:
  project()            projection.py:151-235   (project_scene)
  bin_arrays()         raster/tiles.py:43-79
  blend_forward()      raster/_core.pyx:169-200 (forward_tiles)
  blend_backward()     raster/_core.pyx:315-343 (backward_tiles)
  reduce_slots()       raster/backward.py:70-73 (np.add.at)
  project_backward()   projection.py:255-379   (projection_backward)
  render_forward()     raster/forward.py:37-54
  render_backward()    raster/backward.py:77-99
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libssg_oracle.so")
_lib = None

T_ALIGN = np.diag([1.0, -1.0, -1.0, 1.0])  # camera.py:19
TILE = 16


class OraCam(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3),
                ("campos", ctypes.c_double * 3), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("tan_fovx", ctypes.c_double), ("tan_fovy", ctypes.c_double),
                ("near", ctypes.c_double), ("s", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


def build():
    subprocess.run(["make", "-s", "-C", _HERE, "libssg_oracle.so"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "ssg_oracle.c"))):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.ora_bin_count.restype = ctypes.c_int64
        L.ora_erf.restype = ctypes.c_double
        L.ora_erf.argtypes = [ctypes.c_double]
        L.ora_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def set_num_threads(n: int):
    lib().ora_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().ora_num_threads())


# ---------------------------------------------------------------- camera
def camera(view, s: float) -> OraCam:
    """camera.py:53-75 + projection.py:152-167, computed with numpy exactly as
    the reference does (R_w2c, t_vec bits feed the depth bits)."""
    c2w = np.asarray(view.c2w, dtype=np.float64).reshape(4, 4)
    if view.convention == "opengl":
        c2w = c2w @ T_ALIGN
    fov_y = view.fov_y
    if fov_y is None:
        fov_y = 2.0 * math.atan(math.tan(view.fov_x / 2.0) * view.height / view.width)
    R_cw = c2w[:3, :3]
    eye = c2w[:3, 3]
    R = R_cw.T
    t = -R @ eye
    cam = OraCam()
    cam.R[:] = [float(x) for x in np.ascontiguousarray(R).ravel()]
    cam.t[:] = [float(x) for x in t]
    cam.campos[:] = [float(x) for x in c2w[:3, 3]]
    cam.fx = view.width / (2.0 * math.tan(view.fov_x / 2.0))
    cam.fy = view.height / (2.0 * math.tan(fov_y / 2.0))
    cam.cx = view.width / 2.0
    cam.cy = view.height / 2.0
    cam.tan_fovx = math.tan(view.fov_x / 2.0)
    cam.tan_fovy = math.tan(fov_y / 2.0)
    cam.near = float(getattr(view, "near", 0.01))
    cam.s = float(s)
    cam.width = int(view.width)
    cam.height = int(view.height)
    return cam


def _scene_arrays(scene):
    n = scene.mu.shape[0]
    deg = int(scene.sh_degree)
    K = (deg + 1) ** 2
    return n, deg, dict(
        mu=_f64(scene.mu, (n, 3)), log_scale=_f64(scene.log_scale, (n, 3)),
        rot=_f64(scene.rot, (n, 4)), sh=_f64(np.asarray(scene.sh)[:, :K, :], (n, K, 3)),
        logits=_f64(scene.opacity_logits, (n, 2)), beta=_f64(scene.beta, (n, 3)),
        dir=_f64(scene.dir, (n, 3)))


# ------------------------------------------------------------ the chain
def project(scene, view, s=0.3):
    n, deg, a = _scene_arrays(scene)
    cam = camera(view, s)
    out = SimpleNamespace(
        valid=np.zeros(n, np.uint8), mean2d=np.zeros((n, 2)), depth=np.zeros(n),
        conic=np.zeros((n, 3)), opacity_pair=np.zeros((n, 2)), radius=np.zeros(n),
        comp=np.zeros(n), skew2d=np.zeros((n, 2)), color=np.zeros((n, 3)))
    nf = ctypes.c_int64(0)
    lib().ora_project(ctypes.c_int64(n), ctypes.c_int(deg), _p(a["mu"]), _p(a["log_scale"]),
                      _p(a["rot"]), _p(a["sh"]), _p(a["logits"]), _p(a["beta"]), _p(a["dir"]),
                      ctypes.byref(cam), _p(out.valid), _p(out.mean2d), _p(out.depth),
                      _p(out.conic), _p(out.opacity_pair), _p(out.radius), _p(out.comp),
                      _p(out.skew2d), _p(out.color), ctypes.byref(nf))
    out.valid = out.valid.astype(bool)
    out.n_skew_fallback = int(nf.value)
    return out


def bin_arrays(mean2d, radius, depth, valid, width, height):
    mean2d = _f64(mean2d)
    radius = _f64(radius)
    depth = _f64(depth)
    valid = np.ascontiguousarray(valid, dtype=np.uint8)
    n = mean2d.shape[0]
    ntx, nty = -(-width // TILE), -(-height // TILE)
    counts = np.zeros(n, np.int64)
    M = int(lib().ora_bin_count(ctypes.c_int64(n), _p(mean2d), _p(radius), _p(valid),
                                ctypes.c_int(width), ctypes.c_int(height), _p(counts)))
    inst_prim = np.zeros(M, np.int64)
    inst_tile = np.zeros(M, np.int64)
    ranges = np.zeros((ntx * nty, 2), np.int64)
    rc = lib().ora_bin_fill(ctypes.c_int64(n), _p(mean2d), _p(radius), _p(depth), _p(valid),
                            ctypes.c_int(width), ctypes.c_int(height), ctypes.c_int64(M),
                            _p(inst_prim), _p(inst_tile), _p(ranges))
    if rc != 0:
        raise RuntimeError(f"ora_bin_fill failed ({rc})")
    return SimpleNamespace(tile_px=TILE, tiles_x=ntx, tiles_y=nty, ranges=ranges,
                           inst_prim=inst_prim, inst_tile=inst_tile, counts=counts)


def blend_forward(proj, grid, width, height, background):
    bg = _f64(background, (3,))
    img = np.zeros((height, width, 3))
    final_T = np.zeros((height, width))
    n_contrib = np.zeros((height, width), np.int32)
    last_idx = np.zeros((height, width), np.int64)
    lib().ora_blend_fwd(_p(_f64(proj.mean2d)), _p(_f64(proj.conic)), _p(_f64(proj.skew2d)),
                        _p(_f64(proj.opacity_pair)), _p(_f64(proj.color)), _p(grid.inst_prim),
                        _p(grid.ranges), ctypes.c_int64(grid.ranges.shape[0]),
                        ctypes.c_int(grid.tiles_x), ctypes.c_int(width), ctypes.c_int(height),
                        _p(bg), _p(img), _p(final_T), _p(n_contrib), _p(last_idx))
    return img, final_T, n_contrib, last_idx


def blend_backward(proj, grid, width, height, background, final_T, last_idx, dL):
    bg = _f64(background, (3,))
    M = grid.inst_prim.shape[0]
    slots = np.zeros((M, 12))
    lib().ora_blend_bwd(_p(_f64(proj.mean2d)), _p(_f64(proj.conic)), _p(_f64(proj.skew2d)),
                        _p(_f64(proj.opacity_pair)), _p(_f64(proj.color)), _p(grid.inst_prim),
                        _p(grid.ranges), ctypes.c_int64(grid.ranges.shape[0]), ctypes.c_int64(M),
                        ctypes.c_int(grid.tiles_x), ctypes.c_int(width), ctypes.c_int(height),
                        _p(bg), _p(_f64(final_T)),
                        _p(np.ascontiguousarray(last_idx, dtype=np.int64)), _p(_f64(dL)),
                        _p(slots))
    return slots


def reduce_slots(grid, slots, n):
    out = np.zeros((n, 12))
    lib().ora_reduce_slots(ctypes.c_int64(grid.inst_prim.shape[0]), _p(grid.inst_prim),
                           _p(_f64(slots)), ctypes.c_int64(n), _p(out))
    return out


def project_backward(scene, view, s, screen12):
    n, deg, a = _scene_arrays(scene)
    K = (deg + 1) ** 2
    cam = camera(view, s)
    g = SimpleNamespace(
        d_mu=np.zeros((n, 3)), d_log_scale=np.zeros((n, 3)), d_rot=np.zeros((n, 4)),
        d_sh=np.zeros((n, K, 3)), d_opacity_logits=np.zeros((n, 2)), d_beta=np.zeros((n, 3)),
        d_dir=np.zeros((n, 3)), g_uv=np.zeros(n), g_z=np.zeros(n))
    lib().ora_project_backward(
        ctypes.c_int64(n), ctypes.c_int(deg), _p(a["mu"]), _p(a["log_scale"]), _p(a["rot"]),
        _p(a["sh"]), _p(a["logits"]), _p(a["beta"]), _p(a["dir"]), ctypes.byref(cam),
        _p(_f64(screen12, (n, 12))), _p(g.d_mu), _p(g.d_log_scale), _p(g.d_rot), _p(g.d_sh),
        _p(g.d_opacity_logits), _p(g.d_beta), _p(g.d_dir), _p(g.g_uv), _p(g.g_z))
    return g


def render_forward(scene, view, s=0.3):
    """raster/forward.py:37-54; returns a FrameBundle-like namespace plus the
    intermediate projection and grid (for list parity checks)."""
    W, H = int(view.width), int(view.height)
    if W > 65535 or H > 65535:
        raise ValueError("image dimension overflow")
    proj = project(scene, view, s)
    grid = bin_arrays(proj.mean2d, proj.radius, proj.depth, proj.valid, W, H)
    img, final_T, n_contrib, last_idx = blend_forward(proj, grid, W, H, scene.background)
    return SimpleNamespace(color=img, final_T=final_T, n_contrib=n_contrib, last_idx=last_idx,
                           width=W, height=H, n_primitives=int(scene.mu.shape[0]),
                           n_instances=int(grid.inst_prim.shape[0]), s=s, proj=proj, grid=grid)


def render_backward(scene, view, frame, dL):
    """raster/backward.py:77-99 (recomputes projection + binning like the
    reference).  Returns a GradientBundle-like namespace plus the per-primitive
    screen gradients (screen12) for stage-level parity."""
    W, H = frame.width, frame.height
    dL = _f64(dL)
    proj = project(scene, view, frame.s)
    grid = bin_arrays(proj.mean2d, proj.radius, proj.depth, proj.valid, W, H)
    if grid.inst_prim.shape[0] != frame.n_instances:
        raise ValueError("instance count differs from the forward pass")
    slots = blend_backward(proj, grid, W, H, scene.background, frame.final_T, frame.last_idx, dL)
    n = int(scene.mu.shape[0])
    screen12 = reduce_slots(grid, slots, n)
    g = project_backward(scene, view, frame.s, screen12)
    g.n_skew_fallback = proj.n_skew_fallback
    g.screen12 = screen12
    return g


def erf(x):
    x = _f64(x)
    out = np.zeros_like(x)
    lib().ora_erf_many(ctypes.c_int64(x.size), _p(x), _p(out))
    return out
