"""Pipelined training steps (Trainer(pipelined=True)): no host read-back
inside a step; the finite-loss branch (fit2d.py:70-71) and the instance
capacity check are a device flag consumed by Adam and the interval
statistics, resolved when the next step starts.  The parameters must follow
the synchronous loop: same updates, same skipped steps, same Adam step
count, and an instance overflow re-run with grown buffers."""

import math

import numpy as np
import pytest
import torch

from helpers import random_scene, random_view
from paper_2605_18334_b200.engine import DeviceScene, Engine
from paper_2605_18334_b200.synthetic import fp32_round
from paper_2605_18334_b200.train import DeviceAdam, IntervalStats, TrainConfig, Trainer

pytestmark = pytest.mark.gpu
FIELDS = ("mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir")


def _setup(seed, n=400):
    rng = np.random.default_rng(seed)
    target_scene = fp32_round(random_scene(rng, n, sh_degree=2))
    views = [random_view(rng, 96, 80) for _ in range(3)]
    eng = Engine()
    tds = DeviceScene.from_host(target_scene)
    targets = [eng.forward(tds, v, 0.3).color.clone() for v in views]
    start = target_scene.copy()
    start.mu += rng.normal(size=start.mu.shape) * 0.02
    return fp32_round(start), views, targets


def _run(start, views, targets, pipelined, nan_at=(), shrink_at=None):
    eng = Engine()
    ds = DeviceScene.from_host(start)
    adam = DeviceAdam(ds, TrainConfig())
    stats = IntervalStats(ds.n, eng.device)
    tr = Trainer(eng, ds, adam, pipelined=pipelined)
    losses = []
    for it in range(8):
        tgt = targets[it % 3]
        if it in nan_at:
            tgt = tgt.clone()
            tgt[0, 0, 0] = float("nan")
        if shrink_at is not None and it == shrink_at:
            eng.capacity = 1  # the next sync-free binning overflows
        v, _ = tr.step(views[it % 3], tgt, it, stats=stats)
        losses.append(v)
    tr.flush()
    torch.cuda.synchronize()
    return ds, adam, stats, tr, [float(x) for x in losses]


def _mismatch(a, b):
    """Fraction of parameter elements differing beyond 1e-6 + 1e-4 rel, per field."""
    out = {}
    for f in FIELDS:
        x, y = getattr(a, f).double().flatten(), getattr(b, f).double().flatten()
        out[f] = float(((x - y).abs() > 1e-6 + 1e-4 * y.abs()).float().mean())
        assert float((x - y).abs().max()) <= 8 * 2 * 0.025, f  # bounded by the steps' updates
    return out


def _close(start, views, targets, a, b, **kw):
    """The gradient sums use float atomics, so two runs of the same loop
    differ at the ulp level, and Adam (eps 1e-15) turns a near-zero
    gradient's sign into a full step.  The pipelined loop must be as close to
    the synchronous one as the synchronous loop is to itself."""
    a2 = _run(start, views, targets, False, **kw)
    base, got = _mismatch(a[0], a2[0]), _mismatch(a[0], b[0])
    for f in FIELDS:
        assert got[f] <= max(3 * base[f], 0.03), (f, got[f], base[f])
    # the loss trajectories agree (the loss of an overflowed step is the re-run's)
    la, lb = np.array(a[4]), np.array(b[4])
    fin = np.isfinite(la)
    assert np.array_equal(fin, np.isfinite(lb))
    np.testing.assert_allclose(lb[fin], la[fin], rtol=2e-3)


def test_pipelined_equals_synchronous():
    start, views, targets = _setup(1)
    a = _run(start, views, targets, False)
    b = _run(start, views, targets, True)
    _close(start, views, targets, a, b)
    assert a[1].t == b[1].t == 8
    assert a[2].steps == b[2].steps == 8
    # interval statistics accumulated over the same steps (per-primitive sums
    # carry the runs' ulp-level noise, their total agrees tightly)
    torch.testing.assert_close(a[2].uv_sum.sum(), b[2].uv_sum.sum(), rtol=2e-3, atol=0.0)


def test_pipelined_skips_non_finite_steps_like_synchronous():
    start, views, targets = _setup(2)
    a = _run(start, views, targets, False, nan_at=(2, 5))
    b = _run(start, views, targets, True, nan_at=(2, 5))
    _close(start, views, targets, a, b, nan_at=(2, 5))
    assert a[1].t == b[1].t == 6
    assert a[2].steps == b[2].steps == 6
    assert b[3].skipped_steps == 2
    assert not math.isfinite(b[4][2]) and not math.isfinite(b[4][5])


def test_pipelined_overflow_reruns_the_step():
    start, views, targets = _setup(3)
    a = _run(start, views, targets, False)
    b = _run(start, views, targets, True, shrink_at=4)
    _close(start, views, targets, a, b)
    assert a[1].t == b[1].t == 8
    assert b[2].steps == 8


def test_pipelined_flushes_before_densify():
    """stats.bundle() and densify_and_prune resolve the pending step first:
    the skipped step (non-finite loss just before densification) is not
    counted in the statistics nor in Adam's step count."""
    from paper_2605_18334_b200.densify import densify_and_prune
    start, views, targets = _setup(4)
    eng = Engine()
    ds = DeviceScene.from_host(start)
    cfg = TrainConfig()
    adam = DeviceAdam(ds, cfg)
    stats = IntervalStats(ds.n, eng.device)
    tr = Trainer(eng, ds, adam, pipelined=True)
    for it in range(4):
        tgt = targets[it % 3]
        if it == 3:
            tgt = tgt.clone()
            tgt[1, 1, 1] = float("nan")
        tr.step(views[it % 3], tgt, it, stats=stats)
    b = stats.bundle()  # flushes: step 3 was skipped on the device
    assert stats.steps == 3 and adam.t == 3 and tr.skipped_steps == 1
    rep = densify_and_prune(ds, b, cfg, adam=adam)
    assert rep["n_primitives"] == ds.n
    stats = IntervalStats(ds.n, eng.device)
    for it in range(4, 7):
        tr.step(views[it % 3], targets[it % 3], it, stats=stats)
    tr.flush()
    assert adam.t == 6 and stats.steps == 3
    for f in FIELDS:
        assert bool(torch.isfinite(getattr(ds, f)).all()), f
