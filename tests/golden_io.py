"""Loading helpers for the reference-generated fixtures in tests/golden/."""

from __future__ import annotations

import glob
import os

import numpy as np

from helpers import scene_from_arrays
from paper_2605_18334_b200.camera import CameraView

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


def load(name):
    d = dict(np.load(os.path.join(GOLDEN_DIR, f"{name}.npz")))
    scene = scene_from_arrays(d)
    view = CameraView(d["c2w"], str(d["convention"]), int(d["width"]), int(d["height"]),
                      float(d["fov_x"]))
    return scene, view, float(d["s"]), d


def rel_floor(got, ref, floor_frac=1e-3):
    """|g - r| / max(|r|, floor) with floor = floor_frac * max|r| of the field
    (the both-tiny escape of the reference's oracles.rel_err, oracles.py:72-80)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    floor = floor_frac * max(float(np.max(np.abs(ref))) if ref.size else 0.0, 1e-30)
    return np.abs(got - ref) / np.maximum(np.abs(ref), floor)
