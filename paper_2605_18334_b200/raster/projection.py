"""Projection results on the host (mirror of reference projection.py:29-38,
151-235 outputs and 238-252 project_splat).

project_scene runs the device projection (ssg_preprocess_forward, fp64) and
returns the per-primitive screen quantities the reference's Projected
exposes to callers: valid, mean2d, depth, conic, opacity_pair, radius, comp,
skew2d, color and n_skew_fallback.  Geometry comes back in fp64 bit for bit
as computed on the device (the fp64 twin record); the colour is the fp32 SH
evaluation the blend uses.  project_splat is the single-primitive variant
with the reference's off-screen cull, used by bin_and_sort callers.
"""

from __future__ import annotations

import dataclasses
from types import SimpleNamespace

import numpy as np

from ..camera import CameraView, to_opencv
from ..engine import DeviceScene, default_engine, dropin_serialized


@dataclasses.dataclass
class Conic:
    a: float
    b: float
    c: float


@dataclasses.dataclass
class Skew2D:
    beta_x: float
    beta_y: float


@dataclasses.dataclass
class ScreenSplat:
    """projection.py:29-38."""
    mean2d: np.ndarray
    conic: Conic
    skew2d: Skew2D
    depth: float
    opacity_pair: tuple
    dilation_comp: float
    color: np.ndarray
    radius: float


@dropin_serialized
def project_scene(scene, view: CameraView, s: float = 0.3) -> SimpleNamespace:
    """projection.py:151-235 on the device; fp64 host arrays."""
    eng = default_engine()
    ds = DeviceScene.from_host(scene, eng.device)
    view = to_opencv(view)
    eng.project(ds, view, s)
    n = ds.n
    rec = eng.splat[:n].cpu().numpy()                     # (n, 8) doubles: the fp32 record's bytes
    rec64 = eng.splat64[:n].cpu().numpy()                 # conic a b c, skew x y, o1 o2, comp
    f32 = rec[:, 2:8].view(np.float32)                    # conic a b c, skew x y, o1 o2, r g b, bands
    return SimpleNamespace(
        valid=eng.valid[:n].cpu().numpy().astype(bool), mean2d=rec[:, 0:2].copy(),
        depth=eng.depth[:n].cpu().numpy(), conic=rec64[:, 0:3].copy(), skew2d=rec64[:, 3:5].copy(),
        opacity_pair=rec64[:, 5:7].copy(), comp=rec64[:, 7].copy(), radius=eng.radius[:n].cpu().numpy(),
        color=f32[:, 7:10].astype(np.float64), n_skew_fallback=eng.n_skew_fallback())


def project_splat(g, view: CameraView, s: float = 0.3) -> ScreenSplat | None:
    """projection.py:238-252: None when invalid or when the mean lies more
    than a radius outside the image."""
    from ..scene import Scene
    p = project_scene(Scene.from_primitives([g]), view, s)
    if not p.valid[0]:
        return None
    v = to_opencv(view)
    r = float(p.radius[0])
    mx, my = p.mean2d[0]
    if not (-r <= mx <= v.width + r and -r <= my <= v.height + r):
        return None
    return ScreenSplat(mean2d=p.mean2d[0], conic=Conic(*p.conic[0]), skew2d=Skew2D(*p.skew2d[0]),
                       depth=float(p.depth[0]), opacity_pair=tuple(p.opacity_pair[0]),
                       dilation_comp=float(p.comp[0]), color=p.color[0], radius=r)


__all__ = ["Conic", "Skew2D", "ScreenSplat", "project_scene", "project_splat"]
