"""Forward rendering (drop-in for reference raster/forward.py:37-54).

render_forward(scene, view, s=0.3, backend_name=None) -> FrameBundle with the
reference's fields, shapes and dtypes: colour (H,W,3) f64, final_T (H,W) f64,
n_contrib (H,W) i32, last_idx (H,W) i64 (global sorted-instance index or
-1).  Projection, binning and blending run on the GPU; only the scene upload
and the result download cross the host boundary.
"""

from __future__ import annotations

import dataclasses

import numpy as np
import torch

from ..camera import CameraView, to_opencv
from ..engine import DeviceScene, camera_struct, default_engine, dropin_serialized
from . import backend

MAX_IMAGE_DIM = 65535  # forward.py:21


@dataclasses.dataclass
class FrameBundle:
    color: np.ndarray       # (H,W,3)
    final_T: np.ndarray     # (H,W)
    n_contrib: np.ndarray   # (H,W) int32
    last_idx: np.ndarray    # (H,W) int64, global sorted-instance index, -1 none
    width: int
    height: int
    n_primitives: int
    n_instances: int
    s: float                # screen dilation used; backward must match


def _to_host(t: torch.Tensor, dtype: torch.dtype) -> np.ndarray:
    """Device -> pinned host copy with the boundary dtype conversion done on
    the device first (the host never loops over the data)."""
    src = t.to(dtype)
    dst = torch.empty(src.shape, dtype=dtype, pin_memory=True)
    dst.copy_(src, non_blocking=True)
    return dst


def frame_to_host(f) -> FrameBundle:
    outs = [_to_host(f.color, torch.float64), _to_host(f.final_T, torch.float64),
            _to_host(f.n_contrib, torch.int32), _to_host(f.last_idx, torch.int64)]
    torch.cuda.current_stream().synchronize()
    c, t, nc, li = (o.numpy() for o in outs)
    return FrameBundle(color=c, final_T=t, n_contrib=nc, last_idx=li, width=f.width,
                       height=f.height, n_primitives=f.n_primitives, n_instances=f.n_instances,
                       s=f.s)


@dropin_serialized
def render_forward(scene, view: CameraView, s: float = 0.3,
                   backend_name: str | None = None) -> FrameBundle:
    backend.active_backend(backend_name)
    view = to_opencv(view)
    if view.width > MAX_IMAGE_DIM or view.height > MAX_IMAGE_DIM:
        raise ValueError("image dimension overflow")
    eng = default_engine()
    ds = DeviceScene.from_host(scene, eng.device)
    f = eng.forward(ds, view, s)
    # what a following render_backward of this very frame can reuse (its
    # own check: raster/backward._reusable)
    eng._dropin_state = (ds, bytes(camera_struct(view, s)), float(s), eng._bin_gen)
    return frame_to_host(f)
