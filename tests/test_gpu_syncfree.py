"""Sync-free frames (no instance-count read-back inside a frame): identical
results when the buffers suffice, a detected (not silent) overflow when they
do not, and view batches that recover from it."""

import numpy as np
import pytest
import torch

from helpers import random_scene, random_view
from paper_2605_18334_b200 import _native as N
from paper_2605_18334_b200.engine import DeviceScene, Engine
from paper_2605_18334_b200.synthetic import fp32_round
from paper_2605_18334_b200.views import render_views

pytestmark = pytest.mark.gpu


def _frame(eng, ds, view, sync):
    f = eng.forward(ds, view, 0.3, sync=sync)
    return [t.clone() for t in (f.color, f.final_T, f.n_contrib, f.last_idx)]


def test_sync_free_frame_equals_synchronised():
    rng = np.random.default_rng(2)
    ds = DeviceScene.from_host(fp32_round(random_scene(rng, 3000, sh_degree=2)))
    view = random_view(rng, 160, 96)
    eng = Engine()
    a = _frame(eng, ds, view, True)
    b = _frame(eng, ds, view, False)
    assert eng.instances() == eng.last_m > 0
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def _far(view, k=8.0):
    """The same view direction from k times farther away: every primitive
    covers about one tile, so far fewer instances."""
    import dataclasses
    c2w = view.c2w.copy()
    c2w[:3, 3] *= k
    return dataclasses.replace(view, c2w=c2w)


def test_overflow_is_detected_and_batches_recover():
    rng = np.random.default_rng(3)
    big = fp32_round(random_scene(rng, 4000, sh_degree=1))
    view = random_view(rng, 128, 96)
    ds_big = DeviceScene.from_host(big)
    eng = Engine()
    eng.forward(ds_big, _far(view), 0.3)                      # sizes the buffers for the far view
    m_far = eng.instances()
    assert 0 < m_far and eng.capacity < 45000
    eng.forward(ds_big, view, 0.3, sync=False)                # far more instances than the capacity
    with pytest.raises(N.NativeError):
        eng.instances()
    want = _frame(Engine(), ds_big, view, True)
    got = _frame(eng, ds_big, view, True)                     # the synchronised frame grows the buffers
    for x, y in zip(want, got):
        assert torch.equal(x, y)
    # a batch whose later views overflow re-renders itself synchronised
    eng2 = Engine()
    views = [_far(view), view, random_view(rng, 128, 96)]
    out = render_views(ds_big, views, engine=eng2)
    ref = render_views(ds_big, views, engine=Engine())
    assert torch.equal(out, ref)
