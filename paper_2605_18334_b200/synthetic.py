"""Seeded synthetic workloads for the benchmark configurations.

Generators follow SURVEY.md Appendix B (RNG call order fixed so the
instance counts quoted there are reproducible):
  frustum_scene  G2 / G3 -- configs 2 and 3 (1M primitives, 1920x1080)
  ball_scene     G4 / G5 -- configs 4 and 5 (3M / 2M primitives, 1297x840)
  orbit_views    reference synthetic.py:49-59
Every array field is rounded to fp32 (and handed back as fp64), so the
device's fp32 appearance storage is lossless and the fp64 oracle sees the
same values.
"""

from __future__ import annotations

import math

import numpy as np

from .camera import OPENCV, CameraView, look_at
from .scene import Scene, SkewGaussian


def fp32_round(scene: Scene) -> Scene:
    f = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    return Scene(f(scene.mu), f(scene.log_scale), f(scene.rot), f(scene.sh),
                 f(scene.opacity_logits), f(scene.beta), f(scene.dir),
                 background=f(scene.background), sh_degree=scene.sh_degree)


def _unit(v):
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _skew_override(rng2, log_scale):
    n = log_scale.shape[0]
    u = _unit(rng2.normal(size=(n, 3)))
    eta = u * (rng2.uniform(0.0, 4.0, n) / np.exp(log_scale).max(axis=1))[:, None]
    w = rng2.uniform(0.0, 1.0, n)
    return w[:, None] * eta, (1.0 - w)[:, None] * eta


def frustum_scene(n: int = 1_000_000, seed: int = 0, width: int = 1920, height: int = 1080,
                  fov_x: float = 1.0, plain_fraction: float = 0.0) -> Scene:
    """G2 (config 2); plain_fraction=0.5 gives G3 (config 3: a seeded half of
    the primitives with beta = dir = 0 and tied opacity logits)."""
    rng = np.random.default_rng(seed)
    tx = math.tan(fov_x / 2.0)
    ty = tx * height / width
    z = rng.uniform(2.0, 12.0, n)
    x = rng.uniform(-1.15, 1.15, n) * tx * z
    y = rng.uniform(-1.15, 1.15, n) * ty * z
    q = _unit(rng.normal(size=(n, 4)))
    sh = np.zeros((n, 16, 3))
    sh[:, 0] = rng.uniform(-1.2, 1.2, (n, 3))
    sh[:, 1:] = rng.normal(size=(n, 15, 3)) * 0.05
    logits = rng.normal(size=(n, 2)) * 0.8
    beta = rng.normal(size=(n, 3)) * 0.6
    dirv = rng.normal(size=(n, 3)) * 0.6
    log_scale = rng.uniform(math.log(0.004), math.log(0.03), (n, 3))
    background = rng.uniform(0.0, 1.0, 3)
    beta, dirv = _skew_override(np.random.default_rng(123), log_scale)
    if plain_fraction > 0.0:
        m = np.random.default_rng(7).uniform(0.0, 1.0, n) < plain_fraction
        beta[m] = 0.0
        dirv[m] = 0.0
        logits[m, 1] = logits[m, 0]
    mu = np.stack([x, y, z], axis=1)
    return fp32_round(Scene(mu, log_scale, q, sh, logits, beta, dirv, background=background,
                            sh_degree=3))


def frustum_view(width: int = 1920, height: int = 1080, fov_x: float = 1.0) -> CameraView:
    """The rotated G2 pose: not the identity, so the depth
    order depends on the fp64 camera transform."""
    c2w = look_at([0.3, -0.2, -0.5], [0.05, 0.02, 7.0], convention=OPENCV)
    return CameraView(c2w, OPENCV, width, height, fov_x)


def ball_scene(n: int = 3_000_000, seed: int = 0) -> Scene:
    """G4 (config 4) / G5 (config 5 at n = 2M)."""
    rng = np.random.default_rng(seed)
    d = _unit(rng.normal(size=(n, 3)))
    mu = d * (1.5 * rng.uniform(0.0, 1.0, n) ** (1.0 / 3.0))[:, None]
    q = _unit(rng.normal(size=(n, 4)))
    log_scale = rng.uniform(math.log(0.002), math.log(0.02), (n, 3))
    sh = np.zeros((n, 16, 3))
    sh[:, 0] = rng.uniform(-1.2, 1.2, (n, 3))
    sh[:, 1:] = rng.normal(size=(n, 15, 3)) * 0.05
    logits = rng.normal(size=(n, 2)) * 0.8
    beta, dirv = _skew_override(rng, log_scale)
    background = rng.uniform(0.0, 1.0, 3)
    return fp32_round(Scene(mu, log_scale, q, sh, logits, beta, dirv, background=background,
                            sh_degree=3))


def orbit_views(n: int, radius: float = 4.0, elevation: float = 1.2, width: int = 64,
                height: int = 64, fov_x: float = 0.9) -> list[CameraView]:
    """reference synthetic.py:49-59: n cameras on a circle looking at the origin."""
    views = []
    for k in range(n):
        a = 2.0 * math.pi * k / n
        eye = (radius * math.cos(a), elevation, radius * math.sin(a))
        views.append(CameraView(look_at(eye, (0.0, 0.0, 0.0), convention=OPENCV), OPENCV,
                                width, height, fov_x))
    return views


def homothetic_sample(scene: Scene, view: CameraView, k: int, seed: int = 99):
    """A 1/k-size copy of a frame workload with the same per-pixel depth
    complexity and per-primitive tile footprint: a random 1/k of the
    primitives, scales enlarged by sqrt(k), image (and focal length) shrunk
    by sqrt(k) at the same field of view.  Every stage's work (N, M, pixels,
    pixel x instance pairs) then scales by ~1/k, so CPU timings of the
    sample extrapolate linearly to the full frame.  Used only to bound the
    CPU-baseline runs."""
    rng = np.random.default_rng(seed)
    n = len(scene)
    keep = np.sort(rng.choice(n, size=max(n // k, 1), replace=False))
    g = math.sqrt(k)
    sub = Scene(scene.mu[keep], scene.log_scale[keep] + math.log(g), scene.rot[keep],
                scene.sh[keep], scene.opacity_logits[keep], scene.beta[keep] / g,
                scene.dir[keep] / g, background=scene.background, sh_degree=scene.sh_degree)
    w = max(int(round(view.width / g)), 16)
    h = max(int(round(view.height / g)), 16)
    v = CameraView(view.c2w, view.convention, w, h, view.fov_x)
    return fp32_round(sub), v


# ---- the reference's blob fixture (synthetic.py:22-47), for the trainer tests
BLOB_BACKGROUND = (0.05, 0.05, 0.08)


def _blob(position, color, scale, opacity=0.92) -> SkewGaussian:
    logit = math.log(opacity / (1.0 - opacity))
    sh = np.zeros((1, 3))
    sh[0] = (np.asarray(color, dtype=np.float64) - 0.5) / 0.28209479177387814
    return SkewGaussian(mu=np.asarray(position, dtype=np.float64),
                        log_scale=np.log(np.asarray(scale, dtype=np.float64)),
                        rot=np.array([1.0, 0.0, 0.0, 0.0]), sh=sh, opacity_logits=np.array([logit, logit]),
                        beta=np.zeros(3), dir=np.zeros(3))


def blob_scene() -> Scene:
    """Three coloured, slightly anisotropic blobs (synthetic.py:39-46)."""
    prims = [_blob((-0.7, 0.0, 0.2), (0.85, 0.15, 0.10), (0.42, 0.30, 0.34)),
             _blob((0.6, 0.35, -0.1), (0.12, 0.75, 0.20), (0.30, 0.44, 0.30)),
             _blob((0.1, -0.5, -0.3), (0.15, 0.25, 0.88), (0.36, 0.30, 0.42))]
    return Scene.from_primitives(prims, background=BLOB_BACKGROUND, sh_degree=0)
