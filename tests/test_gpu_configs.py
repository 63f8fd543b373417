"""Config-level GPU checks (BASELINE.json configs 1-4).

* config 3: on skew-free splats (beta = dir = 0, tied logits) the skew kernel
  must equal a plain-3DGS blend bit for bit, and a mixed 50/50 scene matches
  the C oracle;
* configs 2/3 at full size (1M, 1920x1080): size-independent properties --
  instance lists sorted by (tile, depth, primitive id), ranges consistent,
  bundle invariants, backward finite with zero gradient for unseen primitives;
* config 4 (3M, 1297x840, orbit views): the view-batched forward equals
  per-view renders.
"""

import ctypes

import numpy as np
import pytest
import torch

import golden_io as G
from oracle import oracle as O
from paper_2605_18334_b200 import _native as N
from paper_2605_18334_b200.engine import DeviceScene, Engine, grid_dims
from paper_2605_18334_b200.synthetic import (ball_scene, frustum_scene, frustum_view,
                                             homothetic_sample, orbit_views)

pytestmark = pytest.mark.gpu


def _frame_copy(f):
    return [t.clone() for t in (f.color, f.final_T, f.n_contrib, f.last_idx)]


def test_config3_plain_splats_equal_vanilla_3dgs_bitwise():
    scene = frustum_scene(60_000, seed=11, width=480, height=270, plain_fraction=1.0)
    view = frustum_view(480, 270)
    eng = Engine()
    ds = DeviceScene.from_host(scene)
    f = eng.forward(ds, view, 0.3)
    skew_out = _frame_copy(f)
    bg = (ctypes.c_float * 3)(*[float(x) for x in ds.background])
    N.check(N.lib().ssg_test_blend_forward_vanilla(480, 270, bg, eng.splat.data_ptr(), eng.splat64.data_ptr(),
                                                  ctypes.byref(eng._bins_struct()),
                                                  ctypes.byref(eng._frame_struct()),
                                                  torch.cuda.current_stream().cuda_stream), "vanilla")
    torch.cuda.synchronize()
    for a, b in zip(skew_out, (eng.color, eng.final_T, eng.n_contrib, eng.last_idx)):
        assert torch.equal(a, b)


def test_config3_mixed_scene_matches_oracle():
    full = frustum_scene(1_000_000, seed=0, plain_fraction=0.5)
    scene, view = homothetic_sample(full, frustum_view(), 64)  # 15.6k prims, 240x135
    from paper_2605_18334_b200.raster import render_backward, render_forward
    ref = O.render_forward(scene, view)
    fr = render_forward(scene, view)
    assert fr.n_instances == ref.n_instances
    assert np.max(np.abs(fr.color - ref.color)) <= 1e-4
    np.testing.assert_array_equal(fr.n_contrib, ref.n_contrib)
    np.testing.assert_array_equal(fr.last_idx, ref.last_idx)
    dL = np.random.default_rng(1).normal(size=(view.height, view.width, 3))
    g = render_backward(scene, view, fr, dL)
    rg = O.render_backward(scene, view, ref, dL)
    for k in ("d_mu", "d_log_scale", "d_rot", "d_sh", "d_opacity_logits", "d_beta", "g_uv", "g_z"):
        e = G.rel_floor(getattr(g, k), getattr(rg, k))
        assert np.mean(e <= 1e-3) >= 0.999 and e.max() <= 1e-2, k


def _check_lists(eng, n, m, width, height):
    """Instance lists sorted by (tile, depth, id); ranges = the tile histogram."""
    ntx, nty = grid_dims(width, height)
    ip, it, rg = eng.grid(ntx * nty)
    tile = it.long()
    prim = ip.long()
    depth = eng.depth[:n][prim]
    assert bool((tile[1:] >= tile[:-1]).all())
    same = tile[1:] == tile[:-1]
    dd = depth[1:] - depth[:-1]
    assert bool((dd[same] >= 0).all())
    tie = same & (dd == 0)
    assert bool((prim[1:][tie] > prim[:-1][tie]).all())
    r = rg.long()
    cnt = torch.bincount(tile, minlength=ntx * nty)
    assert torch.equal(r[:, 1] - r[:, 0], cnt)
    assert int(r[-1, 1]) == m and int(r[0, 0]) == 0
    return prim


def test_config4_full_size_lists():
    """G4 view 0 at full size (3M primitives: several depth-sort tiles per
    CTA, the flagged-sum scan across them): M equals the reference's count
    and the lists keep their order."""
    scene = ball_scene(3_000_000, seed=0)
    view = orbit_views(64, radius=4.0, elevation=1.2, width=1297, height=840, fov_x=0.9)[0]
    eng = Engine()
    ds = DeviceScene.from_host(scene)
    f = eng.forward(ds, view, 0.3)
    assert f.n_instances == 17_916_589  # SURVEY.md §8(d), G4 view 0
    _check_lists(eng, len(scene), f.n_instances, 1297, 840)


@pytest.mark.parametrize("plain", [0.0, 0.5])
def test_full_size_properties(plain):
    scene = frustum_scene(1_000_000, plain_fraction=plain)
    view = frustum_view()
    eng = Engine()
    ds = DeviceScene.from_host(scene)
    f = eng.forward(ds, view, 0.3)
    m = f.n_instances
    if plain == 0.0:
        assert m == 9_097_352  # SURVEY.md §8(d), measured from the reference on G2
    prim = _check_lists(eng, len(scene), m, 1920, 1080)
    T = f.final_T
    assert float(T.min()) >= 1e-4 * (1 - 0.99) - 1e-7 and float(T.max()) <= 1.0
    assert bool(torch.isfinite(f.color).all())
    li = f.last_idx.long()
    untouched = f.n_contrib == 0
    assert bool((li[untouched] == -1).all()) and bool((T[untouched] == 1.0).all())
    dL = torch.randn(1080, 1920, 3, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    g = eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dL, rebin=False)
    for t in (g.d_mu, g.d_log_scale, g.d_rot, g.d_sh, g.d_opacity_logits, g.d_eta, g.g_uv, g.g_z):
        assert bool(torch.isfinite(t).all())
    seen = torch.zeros(len(scene), dtype=torch.bool, device="cuda")
    seen[prim] = True
    assert bool((g.d_mu[~seen] == 0).all()) and bool((g.g_z[~seen] == 0).all())


def test_config4_view_batch_equals_single_views():
    scene = ball_scene(200_000, seed=3)
    views = orbit_views(20, width=1297, height=840, fov_x=0.9)  # 3 groups of <= 8 views
    eng = Engine()
    ds = DeviceScene.from_host(scene)
    singles = []
    for v in views:
        f = eng.forward(ds, v, 0.3)
        singles.append(f.color.clone())
    from paper_2605_18334_b200.views import render_views
    batch = render_views(ds, views, engine=eng)
    for a, b in zip(singles, batch):
        assert torch.equal(a, b)
    # several engines on their own streams (views overlap): same pixels
    lanes = [eng, Engine(), Engine()]
    for _ in range(2):
        multi = render_views(ds, views, engine=lanes)
        for a, b in zip(singles, multi):
            assert torch.equal(a, b)
