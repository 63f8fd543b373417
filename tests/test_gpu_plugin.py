"""The reference-interface blend plugin (paper_2605_18334_b200.plugin:
forward_tiles / backward_tiles with raster/_core.pyx's signatures) against
the C oracle's restatement of those kernels, on the oracle's own projection
and binning (the reference's backend-equivalence test, test_backends.py:58-96,
with fp32 tolerances)."""

import numpy as np
import pytest

import golden_io as G
from oracle import oracle as O
from paper_2605_18334_b200 import plugin

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["skew_0", "plain_0", "tight_fov_33x17", "frustum_3k_160x96",
                                  "dense_400_96x80", "kat_occluder"])
def test_plugin_matches_oracle_kernels(name):
    scene, view, s, d = G.load(name)
    W, H = view.width, view.height
    p = O.project(scene, view, s)
    g = O.bin_arrays(p.mean2d, p.radius, p.depth, p.valid, W, H)
    args = (p.mean2d, p.conic, p.skew2d, p.opacity_pair, p.color, g.inst_prim, g.ranges, g.tiles_x, W, H,
            scene.background)
    img, T, nc, li = plugin.forward_tiles(*args)
    rimg, rT, rnc, rli = O.blend_forward(p, g, W, H, scene.background)
    assert img.dtype == np.float64 and T.dtype == np.float64
    assert nc.dtype == np.int32 and li.dtype == np.int64
    assert np.max(np.abs(img - rimg)) <= 1e-4
    assert np.max(np.abs(T - rT)) <= 1e-4
    np.testing.assert_array_equal(nc, rnc)
    np.testing.assert_array_equal(li, rli)
    slots = plugin.backward_tiles(*args, rT, rli, d["dL"])
    rslots = O.blend_backward(p, g, W, H, scene.background, rT, rli, d["dL"])
    assert slots.shape == rslots.shape == (g.inst_prim.shape[0], 12)
    e = G.rel_floor(slots, rslots)
    assert np.mean(e <= 1e-3) >= 0.999 and e.max() <= 1e-2


def test_plugin_rejects_overflow_and_mismatch():
    with pytest.raises(ValueError):
        plugin.forward_tiles(np.zeros((0, 2)), np.zeros((0, 3)), np.zeros((0, 2)), np.zeros((0, 2)),
                             np.zeros((0, 3)), np.zeros(0, np.int64), np.zeros((4, 2), np.int64), 2, 32, 33,
                             np.zeros(3))


def test_plugin_empty():
    img, T, nc, li = plugin.forward_tiles(np.zeros((0, 2)), np.zeros((0, 3)), np.zeros((0, 2)),
                                          np.zeros((0, 2)), np.zeros((0, 3)), np.zeros(0, np.int64),
                                          np.zeros((4, 2), np.int64), 2, 32, 32, np.array([0.2, 0.4, 0.6]))
    assert np.allclose(img, [0.2, 0.4, 0.6]) and np.all(T == 1.0) and np.all(li == -1) and np.all(nc == 0)
