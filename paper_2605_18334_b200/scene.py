"""Primitive store (mirror of the reference Scene / SkewGaussian types).

Structure-of-arrays over skew-Gaussian primitives with the reference's field
names, shapes and fp64 host dtype (pkg/src/skewsplat/scene.py:42-164):
mu (N,3), log_scale (N,3), rot (N,4, w x y z), sh (N,K,3), opacity_logits
(N,2), beta (N,3), dir (N,3), background (3,), sh_degree 0..3.  Any object
with these attributes (including the reference's own Scene) is accepted by
the rasterizer.  PLY serialization: ply.py (save_ply / load_ply, and
load_ply_device straight into the device layout).
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class SkewGaussian:
    """One primitive (scene.py:42-63)."""

    mu: np.ndarray
    log_scale: np.ndarray
    rot: np.ndarray
    sh: np.ndarray
    opacity_logits: np.ndarray
    beta: np.ndarray
    dir: np.ndarray

    def __post_init__(self):
        for name in ("mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir"):
            setattr(self, name, np.asarray(getattr(self, name), dtype=np.float64))


class Scene:
    """SoA primitive set plus background colour and SH degree (scene.py:99-164)."""

    ARRAY_FIELDS = ("mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir")

    def __init__(self, mu, log_scale, rot, sh, opacity_logits, beta, dir,
                 background=(0.0, 0.0, 0.0), sh_degree: int | None = None):
        self.mu = np.asarray(mu, dtype=np.float64).reshape(-1, 3)
        n = self.mu.shape[0]
        self.log_scale = np.asarray(log_scale, dtype=np.float64).reshape(n, 3)
        self.rot = np.asarray(rot, dtype=np.float64).reshape(n, 4)
        sh = np.asarray(sh, dtype=np.float64)
        self.sh = sh if sh.ndim == 3 else sh.reshape(n, -1, 3)
        self.opacity_logits = np.asarray(opacity_logits, dtype=np.float64).reshape(n, 2)
        self.beta = np.asarray(beta, dtype=np.float64).reshape(n, 3)
        self.dir = np.asarray(dir, dtype=np.float64).reshape(n, 3)
        self.background = np.asarray(background, dtype=np.float64).reshape(3)
        if sh_degree is None:
            sh_degree = int(round(math.sqrt(self.sh.shape[1]))) - 1
        if (sh_degree + 1) ** 2 != self.sh.shape[1] or not 0 <= sh_degree <= 3:
            raise ValueError(f"sh coefficient count {self.sh.shape[1]} does not "
                             f"match degree {sh_degree}")
        self.sh_degree = sh_degree

    @classmethod
    def empty(cls, sh_degree: int = 0, background=(0.0, 0.0, 0.0)) -> "Scene":
        k = (sh_degree + 1) ** 2
        z = np.zeros((0, 3))
        return cls(z, z, np.zeros((0, 4)), np.zeros((0, k, 3)), np.zeros((0, 2)), z, z,
                   background=background, sh_degree=sh_degree)

    @classmethod
    def from_primitives(cls, prims, background=(0.0, 0.0, 0.0),
                        sh_degree: int | None = None) -> "Scene":
        if not prims:
            return cls.empty(0 if sh_degree is None else sh_degree, background)
        return cls(*(np.stack([getattr(p, f) for p in prims]) for f in cls.ARRAY_FIELDS),
                   background=background, sh_degree=sh_degree)

    def __len__(self) -> int:
        return self.mu.shape[0]

    def save_ply(self, path):
        """scene.py:177-207 (ply.save_ply)."""
        from .ply import save_ply
        save_ply(self, path)

    def primitive(self, i: int) -> SkewGaussian:
        return SkewGaussian(*(getattr(self, f)[i] for f in self.ARRAY_FIELDS))

    def copy(self) -> "Scene":
        return Scene(*(getattr(self, f).copy() for f in self.ARRAY_FIELDS),
                     background=self.background.copy(), sh_degree=self.sh_degree)
