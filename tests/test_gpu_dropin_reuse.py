"""render_backward right after render_forward of the same scene reuses the
engine's binning and blend decisions instead of recomputing them
(raster/backward._pipelined_backward: speculative replay while the scene is
uploaded chunk-wise, gradients downloaded chunk-wise, a bitwise check at the
end; raster/backward._reusable for screen_gradients).  The result must be
bit-identical to the recomputing path, and any change to the scene,
background, camera, s or frame must end on the full path."""

import numpy as np
import pytest

from helpers import random_scene, random_view
from paper_2605_18334_b200.engine import default_engine
from paper_2605_18334_b200.raster import render_backward, render_forward
from paper_2605_18334_b200.raster import backward as RB
from paper_2605_18334_b200.synthetic import fp32_round

pytestmark = pytest.mark.gpu
GRADS = ("d_mu", "d_log_scale", "d_rot", "d_sh", "d_opacity_logits", "d_beta", "d_dir", "g_uv", "g_z")


def _full(scene, view, frame, dL):
    default_engine()._dropin_state = None   # forces the recomputation
    return render_backward(scene, view, frame, dL)


def _same(a, b):
    for k in GRADS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.n_skew_fallback == b.n_skew_fallback


def test_reuse_is_bitwise_the_recomputation(monkeypatch):
    rng = np.random.default_rng(21)
    scene = fp32_round(random_scene(rng, 2500, sh_degree=3))
    view = random_view(rng, 144, 96)
    dL = np.random.default_rng(2).normal(size=(96, 144, 3))
    calls = []
    orig = RB._pipelined_backward
    monkeypatch.setattr(RB, "_pipelined_backward", lambda *a, **k: calls.append(r := orig(*a, **k)) or r)
    fr = render_forward(scene, view)
    fast = render_backward(scene, view, fr, dL)
    assert calls and calls[-1] is not None          # the pipelined reuse path ran
    ref = _full(scene, view, fr, dL)
    _same(fast, ref)
    # screen_gradients' reuse (_reusable) against its recomputation
    fr = render_forward(scene, view)
    a = RB.screen_gradients(scene, view, fr, dL)
    default_engine()._dropin_state = None
    b = RB.screen_gradients(scene, view, fr, dL)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("field", ["mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir", "background"])
def test_late_chunk_change_is_caught(field, monkeypatch):
    """One value of the LAST primitive (the last upload chunk) changed
    between forward and backward: the speculative result is discarded and
    the projection + binning recomputed."""
    rng = np.random.default_rng(23)
    scene = fp32_round(random_scene(rng, 2000, sh_degree=1))
    view = random_view(rng, 96, 64)
    dL = np.random.default_rng(4).normal(size=(64, 96, 3))
    fr = render_forward(scene, view)
    moved = scene.copy()
    a = getattr(moved, field)
    if field == "background":
        a[1] = 1.0 - a[1]
    elif field in ("mu", "log_scale", "rot"):   # fp64 on the device; tiny, keeps the tile lists
        a[-1].flat[0] += 1e-9
    else:                                       # fp32 appearance fields
        a[-1].flat[0] += 0.25
    eng = default_engine()
    binned = []
    orig = eng.project_and_bin
    monkeypatch.setattr(eng, "project_and_bin", lambda *x, **k: binned.append(1) or orig(*x, **k))
    got = render_backward(moved, view, fr, dL)
    assert binned                                   # the change was caught
    monkeypatch.undo()
    _same(got, _full(moved, view, fr, dL))
    # unchanged: no recomputation
    fr = render_forward(scene, view)
    monkeypatch.setattr(eng, "project_and_bin", lambda *x, **k: binned.append(2) or orig(*x, **k))
    render_backward(scene, view, fr, dL)
    assert 2 not in binned


def test_changes_take_the_full_path(monkeypatch):
    rng = np.random.default_rng(22)
    scene = fp32_round(random_scene(rng, 1500, sh_degree=2))
    view = random_view(rng, 96, 80)
    dL = np.random.default_rng(3).normal(size=(80, 96, 3))
    fr = render_forward(scene, view)
    # a changed scene (same shapes): the full path, the new scene's gradients
    moved = scene.copy()
    moved.sh[:, 0] += 0.01
    got = render_backward(moved, view, fr, dL)
    _same(got, _full(moved, view, fr, dL))
    # a changed frame (last_idx edited): the full path
    fr = render_forward(scene, view)
    fr2 = type(fr)(**{**fr.__dict__, "final_T": fr.final_T.copy()})
    fr2.final_T[0, 0] *= 0.5
    got = render_backward(scene, view, fr2, dL)
    _same(got, _full(scene, view, fr2, dL))
    # an engine that binned since: the full path
    fr = render_forward(scene, view)
    render_forward(scene, random_view(rng, 96, 80))
    got = render_backward(scene, view, fr, dL)
    _same(got, _full(scene, view, fr, dL))


def _frame_same(a, b):
    for k in ("color", "final_T", "n_contrib", "last_idx"):
        x, y = getattr(a, k), getattr(b, k)
        assert x.dtype == y.dtype and np.array_equal(x, y), k
    assert (a.n_instances, a.n_primitives, a.width, a.height, a.s) == \
        (b.n_instances, b.n_primitives, b.width, b.height, b.s)


def test_speculative_forward_is_exact():
    """render_forward renders the engine's previous device scene while the
    caller's scene uploads, then compares the two bitwise: the same scene
    gives the non-speculative frame bit for bit; a changed one (any field,
    last primitive only) is re-rendered from the upload."""
    from paper_2605_18334_b200.raster import forward as RF
    rng = np.random.default_rng(31)
    scene = fp32_round(random_scene(rng, 2200, sh_degree=3))
    views = [random_view(rng, 112, 80) for _ in range(3)]
    eng = default_engine()

    def fresh(sc, v):
        eng._dropin_state = None
        return render_forward(sc, v)

    render_forward(scene, views[0])
    eng._spec_skip = 0
    for v in views:                                  # same scene, new cameras: speculation holds
        got = render_forward(scene, v)
        assert eng._spec_skip == 0
        _frame_same(got, fresh(scene, v))
        eng._spec_skip = 0
    for field in ("mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir"):
        render_forward(scene, views[0])
        eng._spec_skip = 0
        moved = scene.copy()
        getattr(moved, field)[-1].flat[0] += 1e-9 if field in ("mu", "log_scale", "rot") else 0.25
        got = render_forward(moved, views[1])
        assert eng._spec_skip == RF._SPEC_BACKOFF, field   # the change was caught
        _frame_same(got, fresh(moved, views[1]))
        # a backward of that frame is the recompute path's
        dL = np.random.default_rng(5).normal(size=(80, 112, 3))
        fr = render_forward(moved, views[1])
        _same(render_backward(moved, views[1], fr, dL), _full(moved, views[1], fr, dL))


def test_pageable_and_pinned_sources_agree():
    """Caller arrays in ordinary (pageable) host memory go through the pinned
    staging ring (hostlink.to_device) in pieces; results equal those from
    pinned arrays, including arrays larger than one staging buffer."""
    import torch
    from paper_2605_18334_b200 import hostlink
    a = np.random.default_rng(3).normal(size=(3 * hostlink.STAGE_BYTES // 8 + 12345,))
    d = hostlink.to_device(a, torch.device("cuda"))
    assert np.array_equal(d.cpu().numpy(), a)
    rng = np.random.default_rng(41)
    scene = fp32_round(random_scene(rng, 1800, sh_degree=3))
    view = random_view(rng, 100, 70)
    dL = np.random.default_rng(6).normal(size=(70, 100, 3))

    def pinned(x):
        t = torch.empty(x.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = x
        return t.numpy()
    pscene = type(scene)(*(pinned(getattr(scene, f)) for f in scene.ARRAY_FIELDS), background=scene.background,
                         sh_degree=scene.sh_degree)
    default_engine()._dropin_state = None
    fa = render_forward(scene, view)
    ga = render_backward(scene, view, fa, dL)
    fb = render_forward(pscene, view)               # speculative on the pageable upload's copy
    gb = render_backward(pscene, view, fb, pinned(dL))
    _frame_same(fa, fb)
    _same(ga, gb)


def test_speculative_forward_instance_overflow_falls_back():
    """A speculative frame runs without the instance-count read-back; a
    view needing more instances than the buffers hold (a much larger image
    after a small one) overflows, is detected by the final read-back and
    rendered again synchronised: the frame equals a fresh render."""
    rng = np.random.default_rng(51)
    scene = fp32_round(random_scene(rng, 3000, sh_degree=1))
    small = random_view(rng, 480, 320, dist=40.0)   # far away: few instances
    big = random_view(rng, 480, 320, dist=2.5)      # same image size, close: many more
    eng = default_engine()
    eng._dropin_state = None
    eng.capacity = 0  # fresh buffers sized by the small frame
    eng._bins_key = None
    render_forward(scene, small)
    eng._spec_skip = 0
    hits = dict(getattr(eng, "_spec_stats", {}))
    got = render_forward(scene, big)
    st = eng._spec_stats
    assert st["forward_misses"] == hits.get("forward_misses", 0) + 1     # overflow: redone
    assert eng._spec_skip == 0                                          # the scene itself was equal
    eng._dropin_state = None
    fresh = render_forward(scene, big)
    _frame_same(got, fresh)
    dL = np.random.default_rng(2).normal(size=(320, 480, 3))
    _same(render_backward(scene, big, got, dL), _full(scene, big, got, dL))
