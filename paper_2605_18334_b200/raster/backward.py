"""Backward rendering (drop-in for reference raster/backward.py:77-99).

Like the reference, the backward pass recomputes projection and binning from
the scene it is given (backward.py:49-53), checks the instance count against
the frame bundle, replays blending back to front from each pixel's last
blended instance, reduces per-instance gradients per primitive and chains
them through the projection.  All of it runs on the GPU.
"""

from __future__ import annotations

import dataclasses

import numpy as np
import torch

from ..camera import CameraView, to_opencv
from ..engine import DeviceScene, default_engine, dropin_serialized
from . import _link, backend
from .forward import FrameBundle  # noqa: F401


class FrameMismatchError(ValueError):
    """The frame bundle was not produced from this scene/view pair."""


@dataclasses.dataclass
class GradientBundle:
    d_mu: np.ndarray              # (N,3)
    d_log_scale: np.ndarray       # (N,3)
    d_rot: np.ndarray             # (N,4)
    d_sh: np.ndarray              # (N,K,3)
    d_opacity_logits: np.ndarray  # (N,2)
    d_beta: np.ndarray            # (N,3)
    d_dir: np.ndarray             # (N,3)
    g_uv: np.ndarray              # (N,) image-plane positional gradient norm
    g_z: np.ndarray               # (N,) |dL/d camera depth|
    n_skew_fallback: int


def _validate(scene, view, frame, dL_dpixels):
    """backward.py:80-88."""
    if (view.width, view.height) != (frame.width, frame.height):
        raise FrameMismatchError("view dimensions differ from the frame bundle")
    if len(scene.mu) != frame.n_primitives:
        raise FrameMismatchError("primitive count differs from the frame bundle")
    dL = np.ascontiguousarray(dL_dpixels, dtype=np.float64)
    if dL.shape != (frame.height, frame.width, 3):
        raise FrameMismatchError(f"dL_dpixels must be ({frame.height}, {frame.width}, 3)")
    return dL


_SCENE_FIELDS = ("mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir")


def _reusable(eng, ds, cam, frame):
    """The engine's last binning and blend decisions are this frame's when
    the last drop-in render_forward on it rendered a scene equal to `ds`
    (bitwise, on the device) from the same camera and s, and nothing has
    binned since: then the recomputation of backward.py:49-53 would
    reproduce them exactly, and the replay can use them directly.  Returns
    the forward's DeviceScene or None."""
    st = getattr(eng, "_dropin_state", None)
    if st is None:
        return None
    fds, cam_bytes, s, gen = st
    if gen != eng._bin_gen or s != float(frame.s) or cam_bytes != bytes(cam) or eng.last_m != frame.n_instances:
        return None
    if fds.n != ds.n or fds.sh_degree != ds.sh_degree or (eng.final_T.shape != (frame.height, frame.width)):
        return None
    if not np.array_equal(fds.background, ds.background):  # the replay starts from the background (:232)
        return None
    if not all(torch.equal(getattr(fds, f), getattr(ds, f)) for f in _SCENE_FIELDS):
        return None
    return fds


def _device_backward(scene, view, frame, dL):
    """Upload, recompute projection + binning (backward.py:49-53), replay.
    The frame and dL_dpixels uploads run on a second stream while the
    recomputed projection and binning (which need only the scene) run.
    When the engine still holds this frame's own forward (same scene bits,
    camera, s, and the frame's final_T / last_idx unchanged), the
    recomputation is skipped: it would reproduce the same lists and
    decisions."""
    from ..engine import camera_struct
    eng = default_engine()
    dev = eng.device
    ds = DeviceScene.from_host(scene, dev)
    main = torch.cuda.current_stream(dev)
    side = eng.lane_stream()
    side.wait_stream(main)
    with torch.cuda.stream(side):
        final_T = _link.to_device(np.ascontiguousarray(frame.final_T, dtype=np.float64), dev).float()
        last_idx = _link.to_device(np.ascontiguousarray(frame.last_idx, dtype=np.int64), dev).int()
        dL_dev = _link.to_device(dL, dev).float()
    cam = camera_struct(view, frame.s)
    fds = _reusable(eng, ds, cam, frame)
    if fds is not None:
        main.wait_stream(side)
        for t in (final_T, last_idx, dL_dev):
            t.record_stream(main)
        if torch.equal(final_T, eng.final_T) and torch.equal(last_idx, eng.last_idx):
            g = eng.backward(fds, view, frame.s, eng.final_T, eng.last_idx, dL_dev, rebin=False,
                             deterministic=True)
            return eng, g
    m = eng.project_and_bin(ds, cam)
    if m != frame.n_instances:
        raise FrameMismatchError("instance count differs from the forward pass")
    main.wait_stream(side)
    for t in (final_T, last_idx, dL_dev):
        t.record_stream(main)
    # the reference's gradients are bit-reproducible: the
    # drop-in uses the deterministic (fixed-order, atomic-free) reduction
    g = eng.backward(ds, view, frame.s, final_T, last_idx, dL_dev, rebin=False, deterministic=True)
    return eng, g


_OUT_FIELDS = ("d_mu", "d_log_scale", "d_rot", "d_sh", "d_opacity_logits", "d_beta", "d_dir", "g_uv", "g_z")


# 8 chunks measured best at config 2 (16.2 ms backward; 6: 16.8, 12: 17.1;
# uploading the small fields whole and only SH in chunks: 17.4)
_PIPE_CHUNKS = 8


def _pipelined_backward(scene, view, frame, dL, chunks: int | None = None):
    """render_backward for the frame of the engine's last drop-in forward,
    with the host link kept busy in both directions.  Returns None when the
    engine's state cannot be this frame's (the caller then takes the
    recompute path).

    The reference recomputes projection + binning from the scene it is given
    (backward.py:49-53); when that scene is bitwise the forward's, the
    recomputation reproduces the forward's lists and decisions, so the replay
    can start on them at once.  Here the replay runs speculatively while the
    scene is uploaded in primitive chunks (host->device); the projection
    backward of chunk i starts when chunk i has landed, and its fp64
    gradients go back (device->host) while later chunks are still coming
    in.  At the end the uploaded scene and frame are compared bitwise with
    the forward's on the device; any difference discards the speculative
    result and reruns the full recompute path on the uploaded scene (the
    result is then exactly the non-speculative one)."""
    from ..engine import camera_struct
    from ..train import bucket_bounds
    eng = default_engine()
    st = getattr(eng, "_dropin_state", None)
    if st is None:
        return None
    fds, cam_bytes, s, gen = st
    cam = camera_struct(view, frame.s)
    n, deg = fds.n, int(scene.sh_degree)
    if (gen != eng._bin_gen or s != float(frame.s) or cam_bytes != bytes(cam) or eng.last_m != frame.n_instances
            or n != len(scene.mu) or n == 0 or fds.sh_degree != deg
            or eng.final_T.shape != (frame.height, frame.width)
            or not np.array_equal(fds.background, np.asarray(scene.background, dtype=np.float64).reshape(3))):
        return None
    K = fds.K
    dev = eng.device
    main = torch.cuda.current_stream(dev)
    up, down = _link.copy_streams(dev)
    srcs = _link.host_fields(scene, n, K)
    pin = {f: _link.is_pinned(a) for f, a in srcs.items()}
    ds = DeviceScene(*(torch.empty_like(getattr(fds, f)) for f in _SCENE_FIELDS), fds.background, deg)
    bounds = bucket_bounds(n, chunks or _PIPE_CHUNKS, align=128)
    # host -> device in the order the device needs it: dL, the scene chunk by
    # chunk, the frame's final_T / last_idx (only for the final comparison)
    up.wait_stream(main)
    with torch.cuda.stream(up):
        # the replay needs only dL (it runs on the forward's own final_T /
        # last_idx, which the frame's are compared with at the end)
        dL_dev = _link.to_device(dL, dev).float()
        ev_dl = torch.cuda.Event()
        ev_dl.record(up)

    def upload(a, b):
        with torch.cuda.stream(up):
            conv = _link.upload_rows(ds, srcs, a, b, dev, pin)
            ev = torch.cuda.Event()
            ev.record(up)
        return ev, conv

    # pinned sources: every chunk queued at once, before the replay (the link
    # is the critical path and must not wait for the host); pageable: one
    # chunk at a time, each after the device work queued so far
    landed = [upload(a, b) for a, b in bounds] if all(pin.values()) else None
    main.wait_event(ev_dl)
    dL_dev.record_stream(main)
    g = eng.backward(fds, view, frame.s, eng.final_T, eng.last_idx, dL_dev, rebin=False, deterministic=True,
                     projection=False)
    outs = {f: _link.host_empty(getattr(g, "d_eta" if f in ("d_beta", "d_dir") else f).shape, torch.float64)
            for f in _OUT_FIELDS}
    for i, (a, b) in enumerate(bounds):
        ev, conv = landed[i] if landed is not None else upload(a, b)
        main.wait_event(ev)
        _link.finish_rows(conv, main)
        eng.projection_backward(ds, cam, g, rows=(a, b))
        eta = g.d_eta[a:b].to(torch.float64)
        pieces = {f: (eta if f in ("d_beta", "d_dir") else getattr(g, f)[a:b].to(torch.float64))
                  for f in _OUT_FIELDS}
        done = torch.cuda.Event()
        done.record(main)
        down.wait_event(done)
        with torch.cuda.stream(down):
            for f, t in pieces.items():
                outs[f][a:b].copy_(t, non_blocking=True)
        for t in pieces.values():
            t.record_stream(down)
    with torch.cuda.stream(up):
        final_T = _link.to_device(np.ascontiguousarray(frame.final_T, dtype=np.float64), dev).float()
        last_idx = _link.to_device(np.ascontiguousarray(frame.last_idx, dtype=np.int64), dev).int()
        ev_frame = torch.cuda.Event()
        ev_frame.record(up)
    main.wait_event(ev_frame)
    for t in (final_T, last_idx):
        t.record_stream(main)
    frame_diff = (final_T.view(torch.int32) != eng.final_T.view(torch.int32)).any() | (last_idx != eng.last_idx).any()
    scene_diff = _link.scenes_differ(ds, fds)
    differs = bool((scene_diff | frame_diff).item())  # synchronises the main stream
    down.synchronize()
    eng._spec_stats = st2 = getattr(eng, "_spec_stats", {"forward_hits": 0, "forward_misses": 0,
                                                         "backward_hits": 0, "backward_misses": 0})
    st2["backward_misses" if differs else "backward_hits"] += 1
    if differs:
        m = eng.project_and_bin(ds, cam)
        if m != frame.n_instances:
            raise FrameMismatchError("instance count differs from the forward pass")
        g = eng.backward(ds, view, frame.s, final_T, last_idx, dL_dev, rebin=False, deterministic=True)
        got = [_host(x) for x in (g.d_mu, g.d_log_scale, g.d_rot, g.d_sh, g.d_opacity_logits,
                                  g.d_eta, g.d_eta, g.g_uv, g.g_z)]
        torch.cuda.current_stream().synchronize()
        outs = dict(zip(_OUT_FIELDS, got))
    n_fb = eng.n_skew_fallback()
    o = {f: t.numpy() for f, t in outs.items()}
    return GradientBundle(**o, n_skew_fallback=n_fb)


def _host(t: torch.Tensor) -> torch.Tensor:
    src = t.to(torch.float64)
    dst = _link.host_empty(src.shape, torch.float64)
    dst.copy_(src, non_blocking=True)
    return dst


@dropin_serialized
def screen_gradients(scene, view: CameraView, frame, dL_dpixels) -> dict:
    """Per-primitive screen-space gradients (mirror of _screen_gradients,
    backward.py:42-74): d_mean2d, d_conic, d_skew2d, d_opair, d_color."""
    view = to_opencv(view)
    dL = _validate(scene, view, frame, dL_dpixels)
    eng, g = _device_backward(scene, view, frame, dL)
    sc = _host(g.screen)
    torch.cuda.current_stream().synchronize()
    sc = sc.numpy()
    return {"d_mean2d": sc[:, 0:2], "d_conic": sc[:, 2:5], "d_skew2d": sc[:, 5:7],
            "d_opair": sc[:, 7:9], "d_color": sc[:, 9:12]}


@dropin_serialized
def render_backward(scene, view: CameraView, frame, dL_dpixels: np.ndarray,
                    backend_name: str | None = None) -> GradientBundle:
    backend.active_backend(backend_name)
    view = to_opencv(view)
    dL = _validate(scene, view, frame, dL_dpixels)
    with _link.drain_on_error(default_engine().device):
        bundle = _pipelined_backward(scene, view, frame, dL)
    if bundle is not None:
        return bundle
    eng, g = _device_backward(scene, view, frame, dL)
    outs = [_host(x) for x in (g.d_mu, g.d_log_scale, g.d_rot, g.d_sh, g.d_opacity_logits,
                                g.d_eta, g.d_eta, g.g_uv, g.g_z)]
    n_fb = eng.n_skew_fallback()  # synchronizes the stream
    torch.cuda.current_stream().synchronize()
    o = [x.numpy() for x in outs]
    return GradientBundle(d_mu=o[0], d_log_scale=o[1], d_rot=o[2], d_sh=o[3],
                          d_opacity_logits=o[4], d_beta=o[5], d_dir=o[6], g_uv=o[7], g_z=o[8],
                          n_skew_fallback=n_fb)
