"""Edge cases through the drop-in API against the C oracle: empty scenes,
scenes entirely behind the camera, images smaller than a tile or not a
multiple of 16, every SH degree (the reference tests these shapes in
test_raster_forward.py / test_raster_backward.py)."""

import numpy as np
import pytest

import golden_io as G
from helpers import random_scene, random_view
from oracle import oracle as O
from paper_2605_18334_b200.raster import render_backward, render_forward
from paper_2605_18334_b200.scene import Scene
from paper_2605_18334_b200.synthetic import fp32_round

pytestmark = pytest.mark.gpu
GRADS = ("d_mu", "d_log_scale", "d_rot", "d_sh", "d_opacity_logits", "d_beta", "d_dir", "g_uv", "g_z")


def _check(scene, view):
    fr = render_forward(scene, view)
    ref = O.render_forward(scene, view)
    assert fr.n_instances == ref.n_instances
    assert np.max(np.abs(fr.color - ref.color), initial=0.0) <= 1e-4
    assert np.max(np.abs(fr.final_T - ref.final_T), initial=0.0) <= 1e-4
    np.testing.assert_array_equal(fr.n_contrib, ref.n_contrib)
    np.testing.assert_array_equal(fr.last_idx, ref.last_idx)
    dL = np.random.default_rng(7).normal(size=(view.height, view.width, 3))
    g = render_backward(scene, view, fr, dL)
    rg = O.render_backward(scene, view, ref, dL)
    for k in GRADS:
        a, b = getattr(g, k), getattr(rg, k)
        assert a.shape == b.shape, k
        if b.size:
            e = G.rel_floor(a, b)
            assert np.mean(e <= 1e-3) >= 0.999 and e.max() <= 1e-2, k
    return fr, g


def test_empty_scene():
    view = random_view(np.random.default_rng(0), 40, 24)
    for deg in (0, 3):
        fr, g = _check(Scene.empty(sh_degree=deg), view)
        assert fr.n_instances == 0
        assert np.all(fr.n_contrib == 0) and np.all(fr.last_idx == -1) and np.all(fr.final_T == 1.0)
        assert g.d_mu.shape == (0, 3) and g.n_skew_fallback == 0


def test_scene_behind_the_camera():
    rng = np.random.default_rng(1)
    view = random_view(rng, 48, 40)
    scene = fp32_round(random_scene(rng, 50, sh_degree=1))
    eye = view.c2w[:3, 3]
    scene.mu = eye + 3.0 * (eye - scene.mu) / np.linalg.norm(eye - scene.mu, axis=1, keepdims=True)
    fr, g = _check(scene, view)
    assert fr.n_instances == 0
    for k in GRADS:
        assert not np.any(getattr(g, k)), k


@pytest.mark.parametrize("wh", [(1, 1), (5, 3), (17, 33), (31, 16)])
def test_tiny_and_ragged_images(wh):
    rng = np.random.default_rng(wh[0] * 100 + wh[1])
    view = random_view(rng, *wh)
    scene = fp32_round(random_scene(rng, 80, sh_degree=2))
    _check(scene, view)


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_every_sh_degree(deg):
    rng = np.random.default_rng(10 + deg)
    view = random_view(rng, 70, 52)
    scene = fp32_round(random_scene(rng, 120, sh_degree=deg))
    _check(scene, view)


@pytest.mark.parametrize("wh", [(30000, 40), (40, 30000), (4100, 2100)])
def test_very_wide_tall_and_large_images(wh):
    """Tile rows / columns far beyond the configs (up to 1875 tiles per row):
    the per-row / per-tile bucket tables of the counting scatter, and splats
    with footprints of 10^4..10^5 pixels.  The north-star bars (the blend's
    decisions are certified, blend.cu)."""
    rng = np.random.default_rng(wh[0] + wh[1])
    view = random_view(rng, *wh, fov_x=1.2)
    scene = fp32_round(random_scene(rng, 300, sh_degree=1))
    fr = render_forward(scene, view)
    ref = O.render_forward(scene, view)
    assert fr.n_instances == ref.n_instances > 0
    assert np.max(np.abs(fr.color - ref.color)) <= 1e-4
    np.testing.assert_array_equal(fr.n_contrib, ref.n_contrib)
    np.testing.assert_array_equal(fr.last_idx, ref.last_idx)
    dL = np.random.default_rng(7).normal(size=(view.height, view.width, 3))
    g = render_backward(scene, view, fr, dL)
    rg = O.render_backward(scene, view, ref, dL)
    for k in GRADS:
        e = G.rel_floor(getattr(g, k), getattr(rg, k))
        assert np.mean(e <= 1e-3) >= 0.999 and e.max() <= 1e-2, (k, float(np.mean(e <= 1e-3)), float(e.max()))
