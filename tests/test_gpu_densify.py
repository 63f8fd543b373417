"""Adaptive density control on the GPU against the
reference's densify_and_prune (optimize/densify.py:24-116) and Adam remap
(optimize/adam.py:99-110), run from oracle/_ref on identical inputs.

Flags, counts, tau_z and every copied value are exact; the moved means of
clones and split children agree to 1e-12 relative (the fp64 exp of the split
half-length may differ from libm's by an ulp)."""

import math
import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from helpers import random_scene
from paper_2605_18334_b200.densify import densify_and_prune
from paper_2605_18334_b200.engine import DeviceScene
from paper_2605_18334_b200.synthetic import fp32_round
from paper_2605_18334_b200.train import DeviceAdam, TrainConfig

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = ("mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir")


def _ref():
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "skewsplat")):
        pytest.skip("oracle/_ref not present")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from skewsplat.optimize.adam import Adam
    from skewsplat.optimize.config import TrainConfig as RefCfg
    from skewsplat.optimize.densify import densify_and_prune as ref_densify
    return Adam, RefCfg, ref_densify


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def _case(seed, n, tau_z=math.nan, radii=False):
    rng = np.random.default_rng(seed)
    scene = fp32_round(random_scene(rng, n, sh_degree=1))
    scene.log_scale[: n // 3] += 1.5  # some large primitives (split candidates)
    scene.opacity_logits[n // 2: n // 2 + n // 10] = -8.0  # some to prune
    g_uv = _f32(rng.uniform(0, 2e-3, n))
    g_z = _f32(rng.uniform(0, 1.0, n))
    d_mu = _f32(rng.normal(size=(n, 3)) * 1e-2)
    z = min(5, n - 1)
    d_mu[z] = 0.0  # a zero clone offset: never cloned
    g_uv[z] = 1.0
    stats = SimpleNamespace(g_uv=g_uv, g_z=g_z.copy(), d_mu=d_mu)
    max_radii = rng.uniform(0, 50, n) if radii else None
    return scene, stats, max_radii


@pytest.mark.parametrize("seed,n,tau_z,radii", [(1, 300, math.nan, False), (2, 1000, 0.7, True),
                                                 (3, 20000, math.nan, False), (4, 5, math.nan, False)])
def test_densify_matches_reference(seed, n, tau_z, radii):
    Adam, RefCfg, ref_densify = _ref()
    scene, stats, max_radii = _case(seed, n, tau_z, radii)
    rcfg, cfg = RefCfg(), TrainConfig()
    for c in (rcfg, cfg):
        c.tau_z = tau_z
        c.max_screen_radius = 30.0 if radii else None
    rng = np.random.default_rng(seed + 100)
    ref_scene = scene.copy()
    radam = Adam(ref_scene, rcfg)
    for f in FIELDS:
        radam.m[f][...] = _f32(rng.normal(size=radam.m[f].shape))
        radam.v[f][...] = _f32(rng.uniform(0, 1, size=radam.v[f].shape))

    ds = DeviceScene.from_host(scene)
    adam = DeviceAdam(ds, cfg)
    names = {"opacity_logits": "logits"}
    for f in FIELDS:
        adam.m[names.get(f, f)].copy_(torch.from_numpy(radam.m[f]).float())
        adam.v[names.get(f, f)].copy_(torch.from_numpy(radam.v[f]).float())
    dstats = SimpleNamespace(g_uv=torch.from_numpy(stats.g_uv).cuda(),
                             g_z=torch.from_numpy(stats.g_z).float().cuda(),
                             d_mu=torch.from_numpy(stats.d_mu).cuda())

    want = ref_densify(ref_scene, stats, rcfg, adam=radam, max_radii=max_radii)
    got = densify_and_prune(ds, dstats, cfg, adam=adam, max_radii=max_radii)
    assert got == want, (got, want)
    assert (math.isnan(cfg.tau_z) and math.isnan(rcfg.tau_z)) or cfg.tau_z == rcfg.tau_z
    assert ds.n == len(ref_scene)
    for f in FIELDS:
        g = getattr(ds, f).double().cpu().numpy().reshape(getattr(ref_scene, f).shape)
        w = getattr(ref_scene, f)
        if f == "mu":
            np.testing.assert_allclose(g, w, rtol=1e-12, atol=1e-15, err_msg=f)
        else:
            np.testing.assert_array_equal(g, _f32(w) if f in ("sh", "opacity_logits", "beta", "dir") else w,
                                          err_msg=f)
        m = adam.m[names.get(f, f)].double().cpu().numpy().reshape(radam.m[f].shape)
        v = adam.v[names.get(f, f)].double().cpu().numpy().reshape(radam.v[f].shape)
        np.testing.assert_array_equal(m, radam.m[f], err_msg="m_" + f)
        np.testing.assert_array_equal(v, radam.v[f], err_msg="v_" + f)
    assert float(dstats.g_z.abs().max()) == 0.0  # densify.py:115


def test_densify_then_render_and_step():
    """The densified scene feeds straight back into the rasterizer and Adam."""
    from helpers import random_view
    from paper_2605_18334_b200.engine import Engine
    from paper_2605_18334_b200.train import Trainer
    scene, stats, _ = _case(7, 400)
    ds = DeviceScene.from_host(scene)
    cfg = TrainConfig()
    adam = DeviceAdam(ds, cfg)
    eng = Engine()
    dstats = SimpleNamespace(g_uv=torch.from_numpy(stats.g_uv).cuda(), g_z=torch.from_numpy(stats.g_z).float().cuda(),
                             d_mu=torch.from_numpy(stats.d_mu).cuda())
    rep = densify_and_prune(ds, dstats, cfg, adam=adam)
    assert rep["n_primitives"] == ds.n != 400
    view = random_view(np.random.default_rng(1), 64, 48)
    tgt = torch.rand((48, 64, 3), device="cuda")
    v, _ = Trainer(eng, ds, adam).step(view, tgt, 0)
    assert math.isfinite(float(v))
