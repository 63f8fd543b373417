"""The C oracle (oracle/ssg_oracle.c) against the reference itself.

Pins the checker before it is trusted: every golden fixture in tests/golden
was produced by the unmodified reference package (tests/golden/make_golden.py),
and when oracle/_ref is importable the oracle is also compared with the live
reference on config 1 (G1).
"""

import os
import sys

import numpy as np
import pytest

import golden_io as G
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", G.names())
def test_oracle_projection_bits_and_lists(name):
    scene, view, s, d = G.load(name)
    f = O.render_forward(scene, view, s)
    p = f.proj
    np.testing.assert_array_equal(p.depth, d["p_depth"])      # bitwise
    np.testing.assert_array_equal(p.mean2d, d["p_mean2d"])    # bitwise
    np.testing.assert_array_equal(p.valid, d["p_valid"])
    for got, ref in ((p.conic, d["p_conic"]), (p.opacity_pair, d["p_opair"]),
                     (p.radius, d["p_radius"]), (p.skew2d, d["p_skew2d"]), (p.color, d["p_color"])):
        if ref.size:
            assert np.max(G.rel_floor(got, ref, 1e-12)) <= 1e-9
    assert p.n_skew_fallback == int(d["n_skew_fallback"])
    assert f.n_instances == int(d["n_instances"])
    np.testing.assert_array_equal(f.grid.inst_prim, d["inst_prim"])
    np.testing.assert_array_equal(f.grid.inst_tile, d["inst_tile"])
    np.testing.assert_array_equal(f.grid.ranges, d["ranges"])


@pytest.mark.parametrize("name", G.names())
def test_oracle_blend_matches_reference(name):
    scene, view, s, d = G.load(name)
    f = O.render_forward(scene, view, s)
    assert np.max(np.abs(f.color - d["color"])) <= 1e-12
    assert np.max(np.abs(f.final_T - d["final_T"])) <= 1e-12
    np.testing.assert_array_equal(f.n_contrib, d["n_contrib"])
    np.testing.assert_array_equal(f.last_idx, d["last_idx"])


@pytest.mark.parametrize("name", G.names())
def test_oracle_backward_matches_reference(name):
    scene, view, s, d = G.load(name)
    f = O.render_forward(scene, view, s)
    g = O.render_backward(scene, view, f, d["dL"])
    for k, lo, hi in (("d_mean2d", 0, 2), ("d_conic", 2, 5), ("d_skew2d", 5, 7),
                      ("d_opair", 7, 9), ("d_color", 9, 12)):
        ref = d["s_" + k]
        if ref.size:
            assert np.max(G.rel_floor(g.screen12[:, lo:hi], ref, 1e-9)) <= 1e-8, k
    for k in ("d_mu", "d_log_scale", "d_rot", "d_sh", "d_opacity_logits", "d_beta", "d_dir",
              "g_uv", "g_z"):
        ref = d["g_" + k]
        if ref.size:
            assert np.max(G.rel_floor(getattr(g, k), ref, 1e-9)) <= 1e-8, k
    assert g.n_skew_fallback == int(d["n_skew_fallback"])


def test_oracle_erf_kats():
    # reference test_kernel_math.py:20-28: erf(0) exact, odd, erf(1)
    assert O.erf(np.array([0.0]))[0] == 0.0
    xs = np.linspace(-6, 6, 241)
    np.testing.assert_array_equal(O.erf(-xs), -O.erf(xs))
    assert abs(O.erf(np.array([1.0]))[0] - 0.8427007929) <= 1e-6
    import math
    assert np.max(np.abs(O.erf(xs) - np.array([math.erf(x) for x in xs]))) <= 1e-13


def test_oracle_empty_scene():
    from helpers import frontal_view
    from paper_2605_18334_b200.scene import Scene
    f = O.render_forward(Scene.empty(background=(0.2, 0.4, 0.6)), frontal_view(48, 32))
    assert np.allclose(f.color, [0.2, 0.4, 0.6]) and np.all(f.final_T == 1.0)
    assert np.all(f.last_idx == -1) and f.n_instances == 0


def _reference():
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "skewsplat")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import skewsplat.raster.forward as rf
        import skewsplat.raster.backward as rb
        from skewsplat.raster import backend
        return rf, rb, backend
    except Exception:  # noqa: BLE001
        return None


def test_oracle_matches_live_reference_on_config1():
    """G1 (config 1: 10k primitives, 256x256) forward + backward, oracle vs
    the reference package itself (skipped where oracle/_ref is absent)."""
    r = _reference()
    if r is None:
        pytest.skip("oracle/_ref (reference build) not present")
    rf, rb, backend = r
    from helpers import random_scene, random_view
    from paper_2605_18334_b200.synthetic import fp32_round
    rng = np.random.default_rng(0)
    scene = fp32_round(random_scene(rng, 10000, sh_degree=2))
    view = random_view(rng, 256, 256)
    ref = rf.render_forward(scene, view, backend_name=backend.active_backend())
    f = O.render_forward(scene, view)
    assert f.n_instances == ref.n_instances == 336948
    assert np.max(np.abs(f.color - ref.color)) <= 1e-12
    np.testing.assert_array_equal(f.last_idx, ref.last_idx)
    np.testing.assert_array_equal(f.n_contrib, ref.n_contrib)
    dL = np.random.default_rng(1).normal(size=(256, 256, 3))
    rg = rb.render_backward(scene, view, ref, dL, backend_name=backend.active_backend())
    g = O.render_backward(scene, view, f, dL)
    for k in ("d_mu", "d_log_scale", "d_rot", "d_sh", "d_opacity_logits", "d_beta", "g_uv", "g_z"):
        assert np.max(G.rel_floor(getattr(g, k), getattr(rg, k), 1e-9)) <= 1e-7, k
