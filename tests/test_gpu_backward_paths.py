"""The engine's backward (ssg_zero_prim_grads on a side stream under the
blend, then ssg_preprocess_backward_ex visiting only primitives with a
non-zero screen gradient) against the plain ssg_preprocess_backward on the
same screen gradients: the projection outputs must be bit-identical."""

import ctypes

import numpy as np
import pytest
import torch

from helpers import random_scene, random_view
from paper_2605_18334_b200 import _native as N
from paper_2605_18334_b200.engine import DeviceScene, Engine, camera_struct
from paper_2605_18334_b200.synthetic import fp32_round

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,deg", [(1, 3), (37, 0), (4000, 2), (25000, 3), (9001, 1)])
def test_ex_backward_equals_plain_pair(n, deg):
    rng = np.random.default_rng(n)
    scene = fp32_round(random_scene(rng, n, sh_degree=deg))
    view = random_view(rng, 200, 120)
    ds = DeviceScene.from_host(scene)
    eng = Engine()
    f = eng.forward(ds, view, 0.3)
    dL = torch.randn(120, 200, 3, device="cuda", generator=torch.Generator("cuda").manual_seed(n))
    outs = lambda g: (g.d_mu, g.d_log_scale, g.d_rot, g.d_sh, g.d_opacity_logits, g.d_eta, g.g_uv, g.g_z)  # noqa: E731
    # poison the outputs: the ex path must overwrite every element
    g0 = eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dL, rebin=False)
    for t in outs(g0):
        t.fill_(float("nan"))
    g = eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dL, rebin=False)
    got = [t.clone() for t in outs(g)]
    for t in got:
        assert bool(torch.isfinite(t).all())
    # the plain projection backward (zero-fills itself) on the same screen sums
    for t in outs(g):
        t.fill_(float("nan"))
    L = N.lib()
    sc, cam, gs = ds.struct(), camera_struct(view, 0.3), eng._grad_struct()
    N.check(L.ssg_preprocess_backward(ctypes.byref(sc), ctypes.byref(cam), ctypes.byref(gs),
                                      torch.cuda.current_stream().cuda_stream), "ssg_preprocess_backward")
    torch.cuda.synchronize()
    for a, b in zip(got, outs(g)):
        assert torch.equal(a, b)
    active = (g.screen != 0).any(dim=1)
    assert bool((g.d_mu[~active] == 0).all()) and bool((g.d_sh[~active] == 0).all())


def test_ex_flags_validated():
    L = N.lib()
    sc = N.SsgScene()
    cam = N.SsgCamera()
    gs = N.SsgGradBuffers()
    sc.n, sc.sh_degree, sc.sh_coeffs = 0, 0, 1
    assert L.ssg_preprocess_backward_ex(ctypes.byref(sc), ctypes.byref(cam), ctypes.byref(gs), 6, None) == \
        N.SSG_ERR_INVALID_ARGUMENT
