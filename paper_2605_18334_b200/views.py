"""View-batched forward rendering (config 4: one scene, many cameras).

The reference renders trajectories one view at a time
(trajectory.py:12-31 loops render_forward); there is no batched call.  Here a
batch of views of one device-resident scene is rendered back to back on one
GPU, each view writing straight into its slice of a (V,H,W,3) output, and
`shard_views` splits a batch across ranks (contiguous blocks, views are
independent, so no collective is needed -- SURVEY.md §8(e)).  On one
engine the projection of each group of up to 8 views is one pass over the
scene (Engine.forward_views / ssg_preprocess_forward_views).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .engine import DeviceScene, Engine, default_engine, dropin_serialized


def shard_views(n_views: int, rank: int, world: int) -> range:
    """Contiguous block of view indices owned by `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def render_views(ds: DeviceScene, views, s: float = 0.3, engine=None,
                 out: torch.Tensor | None = None, check: bool = True) -> torch.Tensor:
    """Forward-render every view of `views` (same width/height) into
    out[v] (float32 (V,H,W,3) on the engine's device).

    `engine` may be one Engine or several: with k engines, the groups of 8
    views go to the engines round-robin, each on its own CUDA stream, so one
    view's latency-bound binning overlaps another view's issue-bound blend
    (the views are independent; every engine owns its buffers).

    check=False: no host round trip at all (no instance-count read-back,
    no capacity check) -- for capturing the batch as a CUDA graph once the
    engines' buffers are sized; the caller then calls instances() on every
    engine after running it (an overflow raises there)."""
    if engine is None:  # the shared default engine: one call at a time
        eng = default_engine()
        with eng.lock:
            return render_views(ds, views, s, engine=eng, out=out, check=check)
    engines = list(engine) if isinstance(engine, (list, tuple)) else [engine]
    eng = engines[0]
    if not views:
        return torch.empty((0, 0, 0, 3), dtype=torch.float32, device=eng.device)
    W, H = int(views[0].width), int(views[0].height)
    if any(int(v.width) != W or int(v.height) != H for v in views):
        raise ValueError("render_views needs views of one image size")
    if out is None:
        out = torch.empty((len(views), H, W, 3), dtype=torch.float32, device=eng.device)
    # every frame after an engine's first skips the instance-count read-back,
    # so the batch runs without host round trips; one check per engine at the
    # end (an overflowing frame makes the batch re-render synchronised)
    if len(engines) == 1:
        # one pass over the scene projects up to MAX_BATCH_VIEWS views
        eng.forward_views(ds, views, s, out=out, sync_first=check)
    else:
        main = torch.cuda.current_stream(eng.device)
        start = torch.cuda.Event()
        start.record(main)
        lanes = [e.lane_stream() for e in engines]
        for st in lanes:
            st.wait_event(start)
        # groups of up to 8 views (one batched projection each), dealt to
        # the engines round-robin
        B = N.MAX_BATCH_VIEWS
        for g, b0 in enumerate(range(0, len(views), B)):
            k = g % len(engines)
            with torch.cuda.stream(lanes[k]):
                engines[k].forward_views(ds, views[b0:b0 + B], s, out=out[b0:b0 + B],
                                         sync_first=check and g < len(engines))
        for st in lanes:
            done = torch.cuda.Event()
            done.record(st)
            main.wait_event(done)
    if not check:
        return out
    used = engines if len(engines) == 1 else engines[:-(-len(views) // N.MAX_BATCH_VIEWS)]
    try:
        for e in used:
            e.instances()
    except N.NativeError:  # capacity overflow somewhere in the batch: redo with read-backs
        for i, v in enumerate(views):
            eng.forward(ds, v, s, color_out=out[i], sync=True)
    return out


_lane_engines: dict = {}


def lane_engines(k: int, device=None) -> list:
    """k engines for render_views on one device (the default engine first),
    cached so their buffers persist across batches."""
    eng = default_engine(device)
    key = str(eng.device)
    lst = _lane_engines.setdefault(key, [eng])
    while len(lst) < k:
        lst.append(Engine(eng.device))
    return lst[:max(k, 1)]


def _views_batch(engines, ds: DeviceScene, views, s: float, u8: bool) -> torch.Tensor:
    """render_views_host's device part: groups of up to 8 views dealt to the
    engines' streams, each group's images copied back on a copy stream as
    soon as it is done.  Returns the (V,H,W,3) host tensor (synchronised)."""
    from .serving import quantize_u8_device
    eng = engines[0]
    W, H, V = int(views[0].width), int(views[0].height), len(views)
    img = torch.empty((V, H, W, 3), dtype=torch.float32, device=eng.device)
    q = torch.empty((V, H, W, 3), dtype=torch.uint8, device=eng.device) if u8 else img
    host = torch.empty((V, H, W, 3), dtype=q.dtype, pin_memory=True)
    main = torch.cuda.current_stream(eng.device)
    start = torch.cuda.Event()
    start.record(main)
    streams = [e.lane_stream() for e in engines]
    copy = getattr(eng, "_copy_stream", None)
    if copy is None:
        copy = eng._copy_stream = torch.cuda.Stream(eng.device)
    for st in streams + [copy]:
        st.wait_event(start)
    B = N.MAX_BATCH_VIEWS
    for g, b0 in enumerate(range(0, V, B)):
        k = g % len(engines)
        b1 = min(V, b0 + B)
        with torch.cuda.stream(streams[k]):
            engines[k].forward_views(ds, views[b0:b1], s, out=img[b0:b1], sync_first=g < len(engines))
            if u8:
                q[b0:b1] = quantize_u8_device(img[b0:b1])
            done = torch.cuda.Event()
            done.record(streams[k])
        copy.wait_event(done)
        with torch.cuda.stream(copy):
            host[b0:b1].copy_(q[b0:b1], non_blocking=True)
    copy.synchronize()
    for st in streams:
        st.synchronize()
    try:
        for e in engines[:-(-V // B)]:
            e.instances()
    except N.NativeError:  # capacity overflow somewhere in the batch: redo synchronised
        out = render_views(ds, views, s, engine=eng)
        return (quantize_u8_device(out) if u8 else out).cpu()
    return host


@dropin_serialized
def render_views_host(scene, views, s: float = 0.3, lanes: int = 4, u8: bool = False):
    """Host API of a view batch (a trajectory, a serving batch): the host
    scene is uploaded once, the views are rendered on the device in groups
    of up to 8 (one batched projection each) dealt round-robin to `lanes`
    engines on their own streams, and every group's images are copied back
    on a copy stream as soon as the group is done (the device-to-host copy
    overlaps the later groups' rendering).  Returns one (V,H,W,3) numpy
    array: float32 colour, or the dataset.py:33-38 u8 quantisation done on
    the device (u8=True, 4x fewer bytes back).

    Serving the same scene batch after batch: the engine keeps the last
    batch's device scene, renders on it while the caller's scene uploads,
    then compares the upload with it bitwise on the device -- equal: the
    images stand (exactly the non-speculative ones); different: the batch is
    rendered again from the upload, which becomes the kept scene."""
    from .raster import _link
    views = list(views)
    engines = lane_engines(lanes)
    eng = engines[0]
    if not views:
        return np.empty((0, 0, 0, 3), dtype=np.uint8 if u8 else np.float32)
    W, H = int(views[0].width), int(views[0].height)
    if any(int(v.width) != W or int(v.height) != H for v in views):
        raise ValueError("render_views needs views of one image size")
    if isinstance(scene, DeviceScene):
        return _views_batch(engines, scene, views, s, u8).numpy()
    prev = getattr(eng, "_host_batch_scene", None)
    n = int(np.asarray(scene.mu).shape[0])
    if (prev is None or n == 0 or prev.n != n or prev.sh_degree != int(scene.sh_degree)
            or not np.array_equal(prev.background, np.asarray(scene.background, dtype=np.float64).reshape(3))):
        ds = DeviceScene.from_host(scene, eng.device)
        eng._host_batch_scene = ds
        return _views_batch(engines, ds, views, s, u8).numpy()
    dev = eng.device
    main = torch.cuda.current_stream(dev)
    up, _ = _link.copy_streams(dev)
    srcs = _link.host_fields(scene, n, prev.K)
    pin = {f: _link.is_pinned(a) for f, a in srcs.items()}
    ds = DeviceScene(*(torch.empty_like(getattr(prev, f)) for f in _link.SCENE_FIELDS), prev.background,
                     prev.sh_degree)
    up.wait_stream(main)
    with torch.cuda.stream(up):
        conv = _link.upload_rows(ds, srcs, 0, n, dev, pin)
        landed = torch.cuda.Event()
        landed.record(up)
    host = _views_batch(engines, prev, views, s, u8)
    main.wait_event(landed)
    _link.finish_rows(conv, main)
    if bool(_link.scenes_differ(ds, prev).item()):
        eng._host_batch_scene = ds
        host = _views_batch(engines, ds, views, s, u8)
    return host.numpy()
