"""Device-resident rasterizer engine (host side of the C ABI).

PyTorch provides device memory and the stream; every computation is a call
into libssg_b200.so.  Buffers are owned here and grown on demand; results
returned by Engine methods are views of engine buffers that stay valid
until the next call with the same engine.

Stage map (reference pkg/src/skewsplat/...):
  Engine.project_and_bin   projection.py:151-235 + raster/tiles.py:43-79
  Engine.forward           raster/forward.py:37-54 (device part)
  Engine.backward          raster/backward.py:77-99 (device part)
"""

from __future__ import annotations

import ctypes
import dataclasses
import functools
import math
import threading

import numpy as np
import torch

from . import _native as N
from .camera import CameraView, intrinsics, to_opencv, world_to_cam

TILE = 16


def grid_dims(width: int, height: int) -> tuple[int, int]:
    """raster/tiles.py:29-30."""
    return -(-width // TILE), -(-height // TILE)


def camera_struct(view: CameraView, s: float) -> N.SsgCamera:
    """Host-side camera constants, evaluated with numpy exactly as the
    reference does (camera.py:60-75, projection.py:152-167)."""
    view = to_opencv(view)
    r_w2c, t_vec = world_to_cam(view)
    K = intrinsics(view)
    cam = N.SsgCamera()
    cam.R[:] = [float(x) for x in np.ascontiguousarray(r_w2c).ravel()]
    cam.t[:] = [float(x) for x in t_vec]
    cam.campos[:] = [float(x) for x in view.c2w[:3, 3]]
    cam.fx, cam.fy = float(K[0, 0]), float(K[1, 1])
    cam.cx, cam.cy = float(K[0, 2]), float(K[1, 2])
    cam.tan_fovx = math.tan(view.fov_x / 2.0)
    cam.tan_fovy = math.tan(view.fov_y / 2.0)
    cam.near_plane = float(view.near)
    cam.s = float(s)
    cam.width, cam.height = int(view.width), int(view.height)
    return cam


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class DeviceScene:
    """Scene resident in HBM: fp64 geometry (mu, log_scale, rot) that decides
    depth order and tile membership, fp32 appearance (sh, logits, beta, dir)."""

    def __init__(self, mu, log_scale, rot, sh, opacity_logits, beta, dir, background, sh_degree):
        self.mu, self.log_scale, self.rot = mu, log_scale, rot
        self.sh, self.opacity_logits, self.beta, self.dir = sh, opacity_logits, beta, dir
        self.background = np.asarray(background, dtype=np.float64).reshape(3)
        self.sh_degree = int(sh_degree)
        self.n = int(mu.shape[0])
        self.K = (self.sh_degree + 1) ** 2

    @classmethod
    def from_host(cls, scene, device=None) -> "DeviceScene":
        """Upload a reference-layout fp64 Scene (any object with the reference
        attributes).  fp64 -> fp32 conversion of the appearance fields runs on
        the device after the copy."""
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        deg = int(scene.sh_degree)
        K = (deg + 1) ** 2
        n = int(np.asarray(scene.mu).shape[0])

        from .hostlink import to_device

        def up(a, shape, f32):
            a = np.ascontiguousarray(a, dtype=np.float64).reshape(shape)
            t = to_device(a, dev)  # pageable sources go through pinned staging
            return t.float() if f32 else t

        sh = np.asarray(scene.sh)
        if sh.ndim != 3:
            sh = sh.reshape(n, -1, 3)
        return cls(up(scene.mu, (n, 3), False), up(scene.log_scale, (n, 3), False),
                   up(scene.rot, (n, 4), False), up(sh[:, :K, :], (n, K, 3), True),
                   up(scene.opacity_logits, (n, 2), True), up(scene.beta, (n, 3), True),
                   up(scene.dir, (n, 3), True), scene.background, deg)

    def rows(self, a: int, b: int) -> "DeviceScene":
        """Primitives [a, b) as a scene of views into this one's storage
        (row slices: the kernels see offset pointers)."""
        return DeviceScene(self.mu[a:b], self.log_scale[a:b], self.rot[a:b], self.sh[a:b],
                           self.opacity_logits[a:b], self.beta[a:b], self.dir[a:b], self.background,
                           self.sh_degree)

    def struct(self) -> N.SsgScene:
        s = N.SsgScene()
        s.n, s.sh_degree, s.sh_coeffs = self.n, self.sh_degree, self.K
        s.mu, s.log_scale, s.rot = _ptr(self.mu), _ptr(self.log_scale), _ptr(self.rot)
        s.sh, s.opacity_logits = _ptr(self.sh), _ptr(self.opacity_logits)
        s.beta, s.dir = _ptr(self.beta), _ptr(self.dir)
        return s


@dataclasses.dataclass
class DeviceFrame:
    color: torch.Tensor       # (H,W,3) f32
    final_T: torch.Tensor     # (H,W) f32
    n_contrib: torch.Tensor   # (H,W) i32
    last_idx: torch.Tensor    # (H,W) i32
    width: int
    height: int
    n_primitives: int
    n_instances: int          # -1 for a sync-free frame (Engine.instances() reads it)
    s: float


@dataclasses.dataclass
class DeviceGrads:
    flat: torch.Tensor        # packed SUM-reducible buffer (see Engine._ensure_grads)
    screen: torch.Tensor      # (N,12)
    d_mu: torch.Tensor
    d_log_scale: torch.Tensor
    d_rot: torch.Tensor
    d_sh: torch.Tensor
    d_opacity_logits: torch.Tensor
    d_eta: torch.Tensor       # d_beta == d_dir (projection.py:365-366)
    g_uv: torch.Tensor
    g_z: torch.Tensor

    SUM_FIELDS = ("d_mu", "d_log_scale", "d_rot", "d_sh", "d_opacity_logits", "d_eta", "g_uv")

    def rows(self, a: int, b: int) -> "DeviceGrads":
        """Primitives [a, b): row slices of every field (flat stays whole)."""
        return DeviceGrads(self.flat, self.screen[a:b], self.d_mu[a:b], self.d_log_scale[a:b], self.d_rot[a:b],
                           self.d_sh[a:b], self.d_opacity_logits[a:b], self.d_eta[a:b], self.g_uv[a:b],
                           self.g_z[a:b])

    def struct(self, d_beta: torch.Tensor | None = None) -> N.SsgGradBuffers:
        g = N.SsgGradBuffers()
        g.screen, g.d_mu, g.d_log_scale = _ptr(self.screen), _ptr(self.d_mu), _ptr(self.d_log_scale)
        g.d_rot, g.d_sh, g.d_opacity_logits = _ptr(self.d_rot), _ptr(self.d_sh), _ptr(self.d_opacity_logits)
        g.d_eta, g.g_uv, g.g_z = _ptr(self.d_eta), _ptr(self.g_uv), _ptr(self.g_z)
        g.d_beta = _ptr(d_beta)
        return g


class Engine:
    def __init__(self, device=None):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.lib = N.lib()
        self._prim_n = -1
        self._bins_key = None
        self._frame_key = None
        self._grad_key = None
        self.capacity = 0
        self.last_m = 0
        self._bin_gen = 0          # bumped by every binning
        self._mask_state = None    # (bin_gen, final_T ptr, last_idx ptr) the blend mask belongs to
        self.blend_mask = None
        # the sorted tile id per instance is output only for introspection
        # (grid(), bin_arrays); throughput loops switch it off
        self.keep_inst_tile = True
        self.stage_events = None  # name -> [(start, end)] CUDA events when enabled
        self.deterministic = False  # backward(): bitwise-repeatable gradients (slower)
        self._exact_pending = None  # event of a deferred forward exact path
        self.all_exact = False      # test mode: every pixel on the exact fp64 path
        # held by the drop-in entry points (dropin_serialized) for a whole call
        self.lock = threading.RLock()

    def _mark(self, name: str):
        """Context for per-stage CUDA-event timing on the launching stream."""
        eng = self

        class _M:
            def __enter__(self):
                if eng.stage_events is not None:
                    self.a = torch.cuda.Event(enable_timing=True)
                    self.a.record()

            def __exit__(self, *exc):
                if eng.stage_events is not None:
                    b = torch.cuda.Event(enable_timing=True)
                    b.record()
                    eng.stage_events.setdefault(name, []).append((self.a, b))
        return _M()

    # ------------------------------------------------------------ buffers
    def _empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=self.device)

    def _ensure_prim(self, n: int):
        if n <= self._prim_n and self._prim_n >= 0:
            return
        nn = max(n, 1)
        self.splat = self._empty((nn, N.SPLAT_BYTES // 8), torch.float64)
        self.splat64 = self._empty((nn, N.SPLAT64_BYTES // 8), torch.float64)
        self.depth_key = self._empty((nn,), torch.int64)
        self.tile_count = self._empty((nn,), torch.int32)
        self.tile_rect = self._empty((nn,), torch.int64)
        self.valid = self._empty((nn,), torch.uint8)
        self.depth = self._empty((nn,), torch.float64)
        self.radius = self._empty((nn,), torch.float64)
        self.n_fallback = self._empty((1,), torch.int32)
        self.depth_order = self._empty((nn,), torch.int32)
        self.rank_offset = self._empty((nn + 1,), torch.int64)
        self.n_inst_dev = torch.zeros((2,), dtype=torch.int64, device=self.device)  # M, running max
        self._prim_n = nn
        self._bins_key = None

    def _prim_struct(self) -> N.SsgPrimBuffers:
        p = N.SsgPrimBuffers()
        p.splat, p.depth_key, p.tile_count = _ptr(self.splat), _ptr(self.depth_key), _ptr(self.tile_count)
        p.tile_rect, p.valid, p.depth = _ptr(self.tile_rect), _ptr(self.valid), _ptr(self.depth)
        p.radius, p.n_skew_fallback = _ptr(self.radius), _ptr(self.n_fallback)
        p.splat64 = _ptr(self.splat64)
        return p

    def _ensure_bins(self, n: int, m: int, W: int, H: int):
        ntx, nty = grid_dims(W, H)
        n_tiles = ntx * nty
        cap = self.capacity
        if m > cap:
            cap = max(int(m * 1.25) + 1024, 1024)
        key = (self._prim_n, cap, W, H)
        if key == self._bins_key:
            return
        if cap != self.capacity:
            self.inst_prim = self._empty((cap,), torch.int32)
            self.inst_tile = self._empty((cap,), torch.int32)
            self.capacity = cap
        words = int(self.lib.ssg_blend_mask_words(cap, max(n_tiles, 1)))
        if self.blend_mask is None or self.blend_mask.numel() < words:
            self.blend_mask = self._empty((words,), torch.int32)
        self.ranges = self._empty((n_tiles, 2), torch.int32)
        if getattr(self, "redo_mask", None) is None or self.redo_mask.numel() < max(n_tiles, 1) * 8:
            self.redo_mask = self._empty((max(n_tiles, 1) * 8,), torch.int32)
        nbytes = ctypes.c_size_t(0)
        N.check(self.lib.ssg_bin_temp_bytes(self._prim_n, cap, W, H, ctypes.byref(nbytes)),
                "ssg_bin_temp_bytes")
        self.temp = self._empty((max(int(nbytes.value), 1),), torch.uint8)
        self._bins_key = key

    def _bins_struct(self) -> N.SsgBinBuffers:
        b = N.SsgBinBuffers()
        b.depth_order, b.rank_offset, b.n_instances = _ptr(self.depth_order), _ptr(self.rank_offset), _ptr(self.n_inst_dev)
        b.capacity = self.capacity
        if self.capacity > 0:
            b.inst_prim = _ptr(self.inst_prim)
            b.inst_tile = _ptr(self.inst_tile) if self.keep_inst_tile else None
        if self._bins_key is not None:
            b.ranges, b.temp, b.temp_bytes = _ptr(self.ranges), _ptr(self.temp), self.temp.numel()
        return b

    def _ensure_frame(self, W: int, H: int):
        if self._frame_key == (W, H):
            return
        self.color = self._empty((H, W, 3), torch.float32)
        self.final_T = self._empty((H, W), torch.float32)
        self.n_contrib = self._empty((H, W), torch.int32)
        self.last_idx = self._empty((H, W), torch.int32)
        self.redo_list = self._empty((max(W * H, 1),), torch.int32)
        self.redo_count = self._empty((1,), torch.int32)
        self._frame_key = (W, H)

    def _frame_struct(self, final_T=None, last_idx=None, color=None, mask=False) -> N.SsgFrameBuffers:
        f = N.SsgFrameBuffers()
        f.blend_mask = _ptr(self.blend_mask) if mask else None
        f.redo_mask, f.redo_list, f.redo_count = _ptr(self.redo_mask), _ptr(self.redo_list), _ptr(self.redo_count)
        f.color, f.n_contrib = _ptr(self.color if color is None else color), _ptr(self.n_contrib)
        f.final_T = _ptr(self.final_T if final_T is None else final_T)
        f.last_idx = _ptr(self.last_idx if last_idx is None else last_idx)
        return f

    def _ensure_grads(self, n: int, K: int):
        """Parameter gradients live in ONE packed f32 buffer, field-major
        [d_mu 3N | d_log_scale 3N | d_rot 4N | d_sh 3KN | d_logits 2N |
        d_eta 3N | g_uv N], so a view-parallel training step reduces them
        with a single SUM all-reduce; g_z (MAX-reduced) is separate."""
        if self._grad_key == (n, K):
            return
        nn = max(n, 1)
        self.g_screen = self._empty((nn, 12), torch.float32)
        widths = (3, 3, 4, 3 * K, 2, 3, 1)
        pad = lambda x: (x + 3) // 4 * 4  # noqa: E731 -- every field 16-byte aligned (float4 access)
        self.g_flat = self._empty((sum(pad(nn * w) for w in widths),), torch.float32)
        views, off = [], 0
        for w in widths:
            views.append(self.g_flat[off:off + nn * w])
            off += pad(nn * w)
        self.g_mu = views[0].view(nn, 3)
        self.g_log_scale = views[1].view(nn, 3)
        self.g_rot = views[2].view(nn, 4)
        self.g_sh = views[3].view(nn, K, 3)
        self.g_logits = views[4].view(nn, 2)
        self.g_eta = views[5].view(nn, 3)
        self.g_uv = views[6].view(nn)
        self.g_z = self._empty((nn,), torch.float32)
        self._grad_key = (n, K)

    def _grad_struct(self) -> N.SsgGradBuffers:
        g = N.SsgGradBuffers()
        g.screen, g.d_mu, g.d_log_scale = _ptr(self.g_screen), _ptr(self.g_mu), _ptr(self.g_log_scale)
        g.d_rot, g.d_sh, g.d_opacity_logits = _ptr(self.g_rot), _ptr(self.g_sh), _ptr(self.g_logits)
        g.d_eta, g.g_uv, g.g_z = _ptr(self.g_eta), _ptr(self.g_uv), _ptr(self.g_z)
        return g

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def lane_stream(self) -> torch.cuda.Stream:
        """This engine's own stream for multi-engine view batches
        (views.render_views): work queued there overlaps other engines'."""
        if getattr(self, "_lane", None) is None:
            self._lane = torch.cuda.Stream(self.device)
        return self._lane

    def _side_stream(self) -> torch.cuda.Stream:
        """Second stream for work that overlaps an issue-bound kernel (the
        projection backward's zero-fill under the blend).  Lowest priority:
        its blocks take the SMs the blend's last wave leaves idle instead of
        displacing blend blocks (a high-priority memset slowed the blend by
        about its own duration)."""
        if getattr(self, "_side", None) is None:
            lo, _ = torch.cuda.Stream.priority_range()
            self._side = torch.cuda.Stream(self.device, priority=lo)
        return self._side

    # ------------------------------------------------------------- stages
    def _bin(self, n: int, W: int, H: int, sync: bool = True) -> int:
        """bin_prepare -> M (one 8-byte D2H) -> bin_finish.  sync=False skips
        the read-back when buffers already exist for this size: the kernels
        stay inside the capacity and instances() detects an overflow later
        (returns -1 for M)."""
        ntx, nty = grid_dims(W, H)
        st = self._stream()
        sync = sync or self.capacity == 0 or self._bins_key is None or self._bins_key[2:] != (W, H) \
            or self._prim_n < n
        self._ensure_bins(n, self.capacity, W, H)
        prim = self._prim_struct()
        with self._mark("bin_prepare"):
            N.check(self.lib.ssg_bin_prepare(n, ctypes.byref(prim), ctypes.byref(self._bins_struct()), st),
                    "ssg_bin_prepare")
        m = int(self.n_inst_dev[0].item()) if sync else -1
        if sync:
            self._ensure_bins(n, m, W, H)
        with self._mark("bin_finish"):
            N.check(self.lib.ssg_bin_finish(n, m, W, H, ctypes.byref(prim), ctypes.byref(self._bins_struct()), st),
                    "ssg_bin_finish")
        self.last_m = m
        self._bin_gen += 1
        return m

    def instances(self, extra: torch.Tensor | None = None):
        """M of the last binning (synchronises); raises if any frame since the
        last call overflowed the instance capacity (those results are
        invalid; the next synchronised binning grows the buffers).  With
        `extra` (a device tensor), its values come back in the same D2H
        read: returns (M, list of floats)."""
        if extra is None:
            m, worst = (int(x) for x in self.n_inst_dev.tolist())
            vals = None
        else:
            host = torch.cat([self.n_inst_dev.double(), extra.double().reshape(-1)]).tolist()
            m, worst, vals = int(host[0]), int(host[1]), host[2:]
        self.n_inst_dev[1] = 0
        if worst > self.capacity:
            self._bins_key = None
            raise N.NativeError(f"sync-free frame needed {worst} instances, capacity {self.capacity}; "
                                "re-run synchronised")
        self.last_m = m
        return m if vals is None else (m, vals)

    def project_and_bin(self, ds: DeviceScene, cam: N.SsgCamera, sync: bool = True) -> int:
        W, H = int(cam.width), int(cam.height)
        if W > 65535 or H > 65535:
            raise ValueError("image dimension overflow")
        self._ensure_prim(ds.n)
        sc = ds.struct()
        with self._mark("preprocess_fwd"):
            N.check(self.lib.ssg_preprocess_forward(ctypes.byref(sc), ctypes.byref(cam),
                                                    ctypes.byref(self._prim_struct()), self._stream()),
                    "ssg_preprocess_forward")
        return self._bin(ds.n, W, H, sync)

    # ------------------------------------------------------- view batches
    _SET_FIELDS = ("splat", "splat64", "depth_key", "tile_count", "tile_rect", "n_fallback")

    def _view_sets(self, k: int) -> list:
        """k per-view screen-record sets for ssg_preprocess_forward_views
        (valid / depth / radius are not written by a batch), grown on demand
        (a short last group reuses the first sets).  Sized like the primary
        buffers (_prim_n rows), so whichever set is bound satisfies
        _ensure_prim's invariant."""
        if getattr(self, "_vsets_n", None) != self._prim_n:
            self._vsets = []
            self._vsets_n = self._prim_n
        nn = self._prim_n
        while len(self._vsets) < k:
            self._vsets.append(dict(splat=self._empty((nn, N.SPLAT_BYTES // 8), torch.float64),
                                    splat64=self._empty((nn, N.SPLAT64_BYTES // 8), torch.float64),
                                    depth_key=self._empty((nn,), torch.int64),
                                    tile_count=self._empty((nn,), torch.int32),
                                    tile_rect=self._empty((nn,), torch.int64),
                                    n_fallback=self._empty((1,), torch.int32)))
        return self._vsets

    @staticmethod
    def _set_struct(d: dict) -> N.SsgPrimBuffers:
        p = N.SsgPrimBuffers()
        p.splat, p.splat64, p.depth_key = _ptr(d["splat"]), _ptr(d["splat64"]), _ptr(d["depth_key"])
        p.tile_count, p.tile_rect, p.n_skew_fallback = _ptr(d["tile_count"]), _ptr(d["tile_rect"]), _ptr(d["n_fallback"])
        p.valid = p.depth = p.radius = None
        return p

    def forward_views(self, ds: DeviceScene, views, s: float = 0.3, out: torch.Tensor | None = None,
                      sync_first: bool = True) -> torch.Tensor:
        """Forward-render a batch of views of one scene (same image size)
        into out[v] (f32 (V,H,W,3)).  The projection runs once per group of
        up to MAX_BATCH_VIEWS views (ssg_preprocess_forward_views: one pass
        over the scene, the view-independent projection part computed once),
        then every view is binned and blended as forward() does.  Outputs
        equal forward() per view bit for bit.  Only the first view reads M
        back (sync_first); the caller checks instances() after the batch.
        Afterwards the engine's screen records are the last view's (a
        backward(rebin=False) of that view is valid)."""
        views = list(views)
        if not views:
            return torch.empty((0, 0, 0, 3), dtype=torch.float32, device=self.device)
        W, H = int(views[0].width), int(views[0].height)
        if any(int(v.width) != W or int(v.height) != H for v in views):
            raise ValueError("forward_views needs views of one image size")
        if W > 65535 or H > 65535:
            raise ValueError("image dimension overflow")
        if out is None:
            out = torch.empty((len(views), H, W, 3), dtype=torch.float32, device=self.device)
        self.finish_exact()
        self._ensure_prim(ds.n)
        sc = ds.struct()
        B = N.MAX_BATCH_VIEWS
        # projection and binning on a high-priority stream, the blends on a
        # low-priority one: when several engines render batches side by side
        # (views.render_views lanes), an engine's latency-bound binning gets
        # the SM slots the other engines' issue-bound blends free up first
        caller = torch.cuda.current_stream(self.device)
        hi, lo = self._prio_streams()
        fork = torch.cuda.Event()
        fork.record(caller)
        hi.wait_event(fork)
        lo.wait_event(fork)
        last_blend = None
        for b0 in range(0, len(views), B):
            chunk = views[b0:b0 + B]
            k = len(chunk)
            cams = [camera_struct(v, s) for v in chunk]
            sets = self._view_sets(k)
            cam_arr = (N.SsgCamera * k)(*cams)
            out_arr = (N.SsgPrimBuffers * k)(*[self._set_struct(d) for d in sets[:k]])
            with torch.cuda.stream(hi):
                if last_blend is not None:  # the view sets are the previous group's blend inputs
                    hi.wait_event(last_blend)
                with self._mark("preprocess_fwd_views"):
                    N.check(self.lib.ssg_preprocess_forward_views(ctypes.byref(sc), cam_arr, out_arr, k,
                                                                  hi.cuda_stream), "ssg_preprocess_forward_views")
            for j, v in enumerate(chunk):
                for f in self._SET_FIELDS:
                    setattr(self, f, sets[j][f])
                W, H = int(cams[j].width), int(cams[j].height)
                with torch.cuda.stream(hi):
                    if last_blend is not None:  # the binning buffers are the previous blend's inputs
                        hi.wait_event(last_blend)
                    m = self._bin(ds.n, W, H, sync_first and b0 + j == 0)
                    binned = torch.cuda.Event()
                    binned.record(hi)
                with torch.cuda.stream(lo):
                    lo.wait_event(binned)
                    self._blend_frame(ds, W, H, m, s, out[b0 + j], False)
                    last_blend = torch.cuda.Event()
                    last_blend.record(lo)
        caller.wait_event(last_blend)
        return out

    def _prio_streams(self):
        if getattr(self, "_prio", None) is None:
            low, high = torch.cuda.Stream.priority_range()
            self._prio = (torch.cuda.Stream(self.device, priority=high), torch.cuda.Stream(self.device, priority=low))
        return self._prio

    def project(self, ds: DeviceScene, view: CameraView, s: float = 0.3) -> torch.Tensor:
        """Projection only (projection.py:151-235): the screen radii (n,)
        fp64 of `view` -- what the reference's densify cadence reads for its
        max_radii (trainer.py:139-141)."""
        cam = camera_struct(view, s)
        if int(cam.width) > 65535 or int(cam.height) > 65535:
            raise ValueError("image dimension overflow")
        self._ensure_prim(ds.n)
        sc = ds.struct()
        N.check(self.lib.ssg_preprocess_forward(ctypes.byref(sc), ctypes.byref(cam),
                                                ctypes.byref(self._prim_struct()), self._stream()),
                "ssg_preprocess_forward")
        self._bin_gen += 1  # the splat records no longer match the last binning
        return self.radius[:ds.n]

    def bin_arrays(self, mean2d, radius, depth, valid, W: int, H: int) -> int:
        """Binning of caller-provided screen arrays (device tensors, fp64/uint8)."""
        n = int(mean2d.shape[0])
        self._ensure_prim(n)
        N.check(self.lib.ssg_bin_rects(n, _ptr(mean2d), _ptr(radius), _ptr(depth), _ptr(valid), W, H,
                                       ctypes.byref(self._prim_struct()), self._stream()),
                "ssg_bin_rects")
        return self._bin(n, W, H)

    def _exact_stream(self) -> torch.cuda.Stream:
        """Stream of the blend's exact path when it overlaps other work."""
        if getattr(self, "_exact", None) is None:
            self._exact = torch.cuda.Stream(self.device)
        return self._exact

    def finish_exact(self):
        """Make the current stream wait for a deferred forward exact path
        (the frame's flagged pixels); no-op when none is pending."""
        if self._exact_pending is not None:
            torch.cuda.current_stream(self.device).wait_event(self._exact_pending)
            self._exact_pending = None

    def forward(self, ds: DeviceScene, view: CameraView, s: float = 0.3,
                color_out: torch.Tensor | None = None, sync: bool = True,
                defer_exact: bool = False, _cam: N.SsgCamera | None = None) -> DeviceFrame:
        """Project, bin and blend one view.  `color_out` (contiguous f32
        (H,W,3) on this device) receives the image instead of the engine's
        own colour buffer (view batches write straight into their slice).
        sync=False: no host round trip inside the frame (see _bin); the
        caller checks instances() before trusting the result.
        defer_exact=True: the exact path over the flagged pixels runs on a
        second stream; the frame is complete only after finish_exact() (a
        following backward() overlaps it with its main kernel)."""
        self.finish_exact()
        if _cam is None:
            cam = camera_struct(view, s)
            W, H = int(cam.width), int(cam.height)
            m = self.project_and_bin(ds, cam, sync)
        else:  # forward_views: the bound screen records are this view's
            cam = _cam
            W, H = int(cam.width), int(cam.height)
            m = self._bin(ds.n, W, H, sync)
        return self._blend_frame(ds, W, H, m, s, color_out, defer_exact)

    def _blend_frame(self, ds: DeviceScene, W: int, H: int, m: int, s: float,
                     color_out: torch.Tensor | None, defer_exact: bool) -> DeviceFrame:
        """The blend half of forward() over the current binning (current stream)."""
        self._ensure_frame(W, H)
        if color_out is not None and (tuple(color_out.shape) != (H, W, 3) or color_out.dtype != torch.float32
                                      or not color_out.is_contiguous() or color_out.device != self.device):
            raise ValueError("color_out must be a contiguous float32 (H, W, 3) tensor on the engine device")
        bg = (ctypes.c_float * 3)(*[float(x) for x in ds.background])
        frame = self._frame_struct(color=color_out, mask=True)
        with self._mark("blend_fwd"):
            if not defer_exact:
                N.check(self.lib.ssg_blend_forward_ex(m, W, H, bg, _ptr(self.splat), _ptr(self.splat64),
                                                      ctypes.byref(self._bins_struct()), ctypes.byref(frame),
                                                      N.SSG_BLEND_ALL_EXACT if self.all_exact else 0,
                                                      self._stream()),
                        "ssg_blend_forward")
            else:
                N.check(self.lib.ssg_blend_forward_ex(m, W, H, bg, _ptr(self.splat), _ptr(self.splat64),
                                                      ctypes.byref(self._bins_struct()), ctypes.byref(frame),
                                                      N.SSG_BLEND_MAIN_ONLY | (N.SSG_BLEND_ALL_EXACT if self.all_exact
                                                                               else 0), self._stream()),
                        "ssg_blend_forward(main)")
        if defer_exact:
            main, ex = torch.cuda.current_stream(self.device), self._exact_stream()
            ev = torch.cuda.Event()
            ev.record(main)
            ex.wait_event(ev)
            N.check(self.lib.ssg_blend_forward_ex(m, W, H, bg, _ptr(self.splat), _ptr(self.splat64),
                                                  ctypes.byref(self._bins_struct()), ctypes.byref(frame),
                                                  N.SSG_BLEND_EXACT_ONLY, ex.cuda_stream),
                    "ssg_blend_forward(exact)")
            self._exact_pending = torch.cuda.Event()
            self._exact_pending.record(ex)
        self._mask_state = (self._bin_gen, _ptr(self.final_T), _ptr(self.last_idx))
        color = self.color if color_out is None else color_out
        return DeviceFrame(color, self.final_T, self.n_contrib, self.last_idx, W, H, ds.n, m, s)

    def _regen_decisions(self, ds: DeviceScene, m: int, W: int, H: int, bg):
        """Re-run the forward blend into scratch buffers for the current
        binning: it rewrites the decision records the backward reads (blend
        mask, exact-path pixel set).  Needed when the caller's frame did not
        come from this engine's last forward over this binning (e.g. the
        drop-in render_backward, which recomputes binning like the
        reference); the decisions are the reference's, so they agree with
        any exact forward of the same scene and view."""
        if getattr(self, "_scratch_key", None) != (W, H):
            self._scratch = [self._empty((H, W, 3), torch.float32), self._empty((H, W), torch.float32),
                             self._empty((H, W), torch.int32), self._empty((H, W), torch.int32)]
            self._scratch_key = (W, H)
        c, t, nc, li = self._scratch
        f = self._frame_struct(final_T=t, last_idx=li, color=c, mask=True)
        f.n_contrib = _ptr(nc)
        N.check(self.lib.ssg_blend_forward_ex(m, W, H, bg, _ptr(self.splat), _ptr(self.splat64),
                                              ctypes.byref(self._bins_struct()), ctypes.byref(f),
                                              N.SSG_BLEND_ALL_EXACT if self.all_exact else 0, self._stream()),
                "ssg_blend_forward (decision records)")

    def backward(self, ds: DeviceScene, view: CameraView, s: float, final_T: torch.Tensor,
                 last_idx: torch.Tensor, dL: torch.Tensor, rebin: bool = True,
                 expect_m: int | None = None, deterministic: bool | None = None,
                 projection: bool = True) -> DeviceGrads:
        """Blend backward + projection backward.  With rebin=True the
        projection and binning are recomputed first (raster/backward.py:49-53)
        and `expect_m` is checked against the new instance count.
        deterministic (default: self.deterministic): bitwise-repeatable
        gradients via ssg_blend_backward_det -- per-(primitive,
        tile) sums combined in a fixed order, no atomics.
        projection=False stops after the screen-space gradients (and the
        zero-fill of the parameter gradients): the caller runs
        projection_backward itself, e.g. over primitive ranges whose
        all-reduce overlaps the next range (train.Trainer buckets)."""
        cam = camera_struct(view, s)
        W, H = int(cam.width), int(cam.height)
        if rebin:
            m = self.project_and_bin(ds, cam)
        else:
            m = self.last_m
        if expect_m is not None and m != expect_m:
            from .raster.backward import FrameMismatchError
            raise FrameMismatchError("instance count differs from the forward pass")
        det = self.deterministic if deterministic is None else deterministic
        if det and m < 0:
            m = self.instances()
        # a deferred forward exact path overlaps this backward's main kernel
        # only when the frame is that forward's own
        mask_ok = self._mask_state == (self._bin_gen, _ptr(final_T), _ptr(last_idx))
        overlap = self._exact_pending is not None and mask_ok and not det
        if not overlap:
            self.finish_exact()
        self._ensure_frame(W, H)
        self._ensure_grads(ds.n, ds.K)
        bg = (ctypes.c_float * 3)(*[float(x) for x in ds.background])
        st = self._stream()
        gs = self._grad_struct()
        # the forward's decision records (blend mask, exact-path pixels)
        # belong to the binning and frame buffers that forward wrote
        if not mask_ok:
            self._regen_decisions(ds, m, W, H, bg)
        # the projection backward's zero-fill runs on a second stream under
        # the issue-bound blend, which leaves DRAM idle; the
        # projection backward then visits only primitives with a non-zero
        # screen gradient.  The side stream starts after everything queued so
        # far (earlier readers of the gradient buffers) and the projection
        # backward waits for it.
        main = torch.cuda.current_stream(self.device)
        side = self._side_stream()
        ev_start, ev_zero = torch.cuda.Event(), torch.cuda.Event()
        ev_start.record(main)
        side.wait_event(ev_start)
        N.check(self.lib.ssg_zero_prim_grads(ds.n, ds.K, ctypes.byref(gs), side.cuda_stream), "ssg_zero_prim_grads")
        ev_zero.record(side)
        frame = self._frame_struct(final_T, last_idx, mask=True)
        with self._mark("blend_bwd"):
            if det:
                nb = int(self.lib.ssg_blend_det_temp_bytes(ds.n, max(m, 0)))
                if getattr(self, "_det_temp", None) is None or self._det_temp.numel() < nb:
                    self._det_temp = self._empty((max(nb, 1),), torch.uint8)
                N.check(self.lib.ssg_blend_backward_det(ds.n, m, W, H, bg, _ptr(self.splat), _ptr(self.splat64),
                                                        ctypes.byref(self._prim_struct()),
                                                        ctypes.byref(self._bins_struct()), ctypes.byref(frame),
                                                        _ptr(dL), ctypes.byref(gs), _ptr(self._det_temp),
                                                        self._det_temp.numel(), st),
                        "ssg_blend_backward_det")
            elif not overlap:
                N.check(self.lib.ssg_blend_backward(ds.n, m, W, H, bg, _ptr(self.splat), _ptr(self.splat64),
                                                    ctypes.byref(self._bins_struct()), ctypes.byref(frame),
                                                    _ptr(dL), ctypes.byref(gs), st),
                        "ssg_blend_backward")
            else:
                # exact half on the exact stream (after the forward's exact
                # half, which is already queued there), main half here
                N.check(self.lib.ssg_zero_screen_grads(ds.n, ctypes.byref(gs), st), "ssg_zero_screen_grads")
                ex = self._exact_stream()
                ev = torch.cuda.Event()
                ev.record(main)
                ex.wait_event(ev)
                N.check(self.lib.ssg_blend_backward_ex(ds.n, m, W, H, bg, _ptr(self.splat), _ptr(self.splat64),
                                                       ctypes.byref(self._bins_struct()), ctypes.byref(frame),
                                                       _ptr(dL), ctypes.byref(gs),
                                                       N.SSG_BLEND_EXACT_ONLY | N.SSG_BLEND_NO_ZERO, ex.cuda_stream),
                        "ssg_blend_backward(exact)")
                N.check(self.lib.ssg_blend_backward_ex(ds.n, m, W, H, bg, _ptr(self.splat), _ptr(self.splat64),
                                                       ctypes.byref(self._bins_struct()), ctypes.byref(frame),
                                                       _ptr(dL), ctypes.byref(gs),
                                                       N.SSG_BLEND_MAIN_ONLY | N.SSG_BLEND_NO_ZERO, st),
                        "ssg_blend_backward(main)")
                done = torch.cuda.Event()
                done.record(ex)
                main.wait_event(done)
                self._exact_pending = None
        main.wait_event(ev_zero)
        n = ds.n
        grads = DeviceGrads(self.g_flat, self.g_screen[:n], self.g_mu[:n], self.g_log_scale[:n], self.g_rot[:n],
                            self.g_sh[:n], self.g_logits[:n], self.g_eta[:n], self.g_uv[:n], self.g_z[:n])
        if projection:
            with self._mark("preprocess_bwd"):
                self.projection_backward(ds, cam, grads)
        return grads

    def projection_backward(self, ds: DeviceScene, cam: N.SsgCamera, grads: DeviceGrads,
                            rows: tuple | None = None) -> None:
        """projection_backward (projection.py:255-379) for primitives
        [a, b) = rows (default: all), from the screen-space gradients of
        `grads` into its parameter fields; only primitives with a non-zero
        screen gradient are visited (the rest were zero-filled by
        backward()).  Range bounds on 128-primitive multiples keep every
        row 16-byte aligned."""
        if rows is not None:
            ds, grads = ds.rows(*rows), grads.rows(*rows)
        sc, gs = ds.struct(), grads.struct()
        N.check(self.lib.ssg_preprocess_backward_ex(ctypes.byref(sc), ctypes.byref(cam), ctypes.byref(gs),
                                                    N.SSG_PREP_BWD_ACTIVE_ONLY, self._stream()),
                "ssg_preprocess_backward_ex")

    def redo_pixels(self) -> int:
        """Pixels of the last forward decided on the exact fp64 path
        (synchronises)."""
        return int(self.redo_count.item())

    # ------------------------------------------------------ introspection
    def grid(self, n_tiles: int):
        """Sorted instance lists and ranges of the last binning (device)."""
        m = self.last_m if self.last_m >= 0 else self.instances()
        if not self.keep_inst_tile:
            raise RuntimeError("this engine does not keep inst_tile (keep_inst_tile = False)")
        return (self.inst_prim[:m], self.inst_tile[:m], self.ranges[:n_tiles])

    def n_skew_fallback(self) -> int:
        return int(self.n_fallback.item())


_engines: dict = {}
_engines_lock = threading.Lock()


def default_engine(device=None) -> Engine:
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = str(dev)
    with _engines_lock:
        if key not in _engines:
            _engines[key] = Engine(dev)
        return _engines[key]


def dropin_serialized(fn):
    """The drop-in entry points share one engine per device (its buffers,
    streams and the last forward's state).  The reference's functions are
    pure and may be called from any thread (SURVEY.md section 8(b),
    threading), so each call holds the current device's default-engine lock
    for its whole duration: concurrent calls run one after another, each
    with the single-thread result."""
    @functools.wraps(fn)
    def call(*args, **kwargs):
        if not torch.cuda.is_available():  # fn's own argument checks, then its CUDA error
            return fn(*args, **kwargs)
        with default_engine().lock:
            return fn(*args, **kwargs)
    return call
