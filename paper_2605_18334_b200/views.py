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

import torch

from . import _native as N
from .engine import DeviceScene, Engine, default_engine


def shard_views(n_views: int, rank: int, world: int) -> range:
    """Contiguous block of view indices owned by `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def render_views(ds: DeviceScene, views, s: float = 0.3, engine=None,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """Forward-render every view of `views` (same width/height) into
    out[v] (float32 (V,H,W,3) on the engine's device).

    `engine` may be one Engine or several: with k engines, the groups of 8
    views go to the engines round-robin, each on its own CUDA stream, so one
    view's latency-bound binning overlaps another view's issue-bound blend
    (the views are independent; every engine owns its buffers)."""
    engines = list(engine) if isinstance(engine, (list, tuple)) else [engine or default_engine()]
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
        eng.forward_views(ds, views, s, out=out, sync_first=True)
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
                engines[k].forward_views(ds, views[b0:b0 + B], s, out=out[b0:b0 + B], sync_first=g < len(engines))
        for st in lanes:
            done = torch.cuda.Event()
            done.record(st)
            main.wait_event(done)
    used = engines if len(engines) == 1 else engines[:-(-len(views) // N.MAX_BATCH_VIEWS)]
    try:
        for e in used:
            e.instances()
    except N.NativeError:  # capacity overflow somewhere in the batch: redo with read-backs
        for i, v in enumerate(views):
            eng.forward(ds, v, s, color_out=out[i], sync=True)
    return out
