"""Config-5 training step on the GPU: the device Adam against the
reference's own Adam (optimize/adam.py, from oracle/_ref) on identical
inputs, and a few view-parallel steps reducing the loss."""

import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from helpers import random_scene, random_view
from paper_2605_18334_b200.engine import DeviceScene, Engine
from paper_2605_18334_b200.synthetic import fp32_round
from paper_2605_18334_b200.train import DeviceAdam, TrainConfig as DevCfg, training_step

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _reference_adam():
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "skewsplat")):
        pytest.skip("oracle/_ref not present")
    sys.path.insert(0, ref)
    from skewsplat.optimize.adam import Adam
    from skewsplat.optimize.config import TrainConfig
    return Adam, TrainConfig


def test_device_adam_matches_reference_adam():
    Adam, TrainConfig = _reference_adam()
    rng = np.random.default_rng(4)
    scene = fp32_round(random_scene(rng, 300, sh_degree=2))
    n, K = len(scene), 9
    g = SimpleNamespace(**{k: rng.normal(size=s).astype(np.float32).astype(np.float64) for k, s in
                           (("d_mu", (n, 3)), ("d_log_scale", (n, 3)), ("d_rot", (n, 4)), ("d_sh", (n, K, 3)),
                            ("d_opacity_logits", (n, 2)), ("d_eta", (n, 3)))})
    g.d_mu[5, 1] = np.nan          # a non-finite row is skipped (adam.py:75-79)
    g.d_beta = g.d_dir = g.d_eta
    scene.rot[7] = [1e-14, 0, 0, 0]  # degenerate quaternion -> identity
    eng = Engine()
    ds = DeviceScene.from_host(scene)
    adam = DeviceAdam(ds, DevCfg())
    ref_scene = scene.copy()
    ref = Adam(ref_scene, TrainConfig())
    for it in range(3):
        eng._ensure_grads(n, K)
        for k, t in (("d_mu", eng.g_mu), ("d_log_scale", eng.g_log_scale), ("d_rot", eng.g_rot),
                     ("d_sh", eng.g_sh), ("d_opacity_logits", eng.g_logits), ("d_eta", eng.g_eta)):
            t.copy_(torch.from_numpy(getattr(g, k)).float())
        grads = SimpleNamespace(d_mu=eng.g_mu, d_log_scale=eng.g_log_scale, d_rot=eng.g_rot, d_sh=eng.g_sh,
                                d_opacity_logits=eng.g_logits, d_eta=eng.g_eta)
        adam.step(grads, it)
        ref.step(ref_scene, g, it)
    assert adam.n_skipped == ref.n_skipped == 3
    for f, dev in (("mu", ds.mu), ("log_scale", ds.log_scale), ("rot", ds.rot), ("sh", ds.sh),
                   ("opacity_logits", ds.opacity_logits), ("beta", ds.beta), ("dir", ds.dir)):
        got = dev.double().cpu().numpy()
        want = getattr(ref_scene, f)
        np.testing.assert_allclose(got, want, rtol=2e-6, atol=2e-6, err_msg=f)


def test_training_steps_reduce_loss():
    rng = np.random.default_rng(8)
    target_scene = fp32_round(random_scene(rng, 60, sh_degree=1))
    view = random_view(rng, 64, 64)
    eng = Engine()
    tgt = eng.forward(DeviceScene.from_host(target_scene), view, 0.3).color.clone()
    start = target_scene.copy()
    start.mu += rng.normal(size=start.mu.shape) * 0.05
    ds = DeviceScene.from_host(fp32_round(start))
    adam = DeviceAdam(ds, DevCfg(lr_position=5e-3, lambda_ssim=0.0))
    losses = [float(training_step(eng, ds, adam, view, tgt)) for _ in range(40)]
    assert losses[-1] < 0.7 * losses[0], losses[::8]
