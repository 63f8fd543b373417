"""Concurrent first calls: the per-device one-time setup (function attributes,
the SSIM window in __constant__ memory, the cooperative sort's grid size) is
guarded per device ordinal, so host threads that hit it together in a fresh
process (ctypes drops the GIL around every ABI call) all get the same results
as one thread."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, threading
import numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from helpers import random_scene, random_view
from paper_2605_18334_b200.engine import DeviceScene, Engine
from paper_2605_18334_b200.synthetic import fp32_round
from paper_2605_18334_b200.train import ImageLoss

rng = np.random.default_rng(2)
scene = fp32_round(random_scene(rng, 3000, sh_degree=3))
views = [random_view(rng, 96, 64) for _ in range(6)]
dL = torch.from_numpy(np.random.default_rng(3).normal(size=(64, 96, 3))).float()
target = torch.from_numpy(np.random.default_rng(4).uniform(size=(64, 96, 3))).float()

def work(view, out, det):
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        eng = Engine()
        ds = DeviceScene.from_host(scene)
        f = eng.forward(ds, view, 0.3)
        g = eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dL.cuda(), rebin=False, deterministic=det)
        loss = ImageLoss(96, 64, 0.2, eng.device)
        d = loss(f.color, target.cuda())
        s.synchronize()
        out.append((f.color.cpu(), g.flat.cpu() if det else None, d.cpu(), loss.value_tensor().cpu()))

res = [[] for _ in views]
ts = [threading.Thread(target=work, args=(v, res[i], True)) for i, v in enumerate(views)]
for t in ts: t.start()
for t in ts: t.join()
ref = [[] for _ in views]
for i, v in enumerate(views):
    work(v, ref[i], True)
for a, b in zip(res, ref):
    assert len(a) == 1 and len(b) == 1
    for x, y in zip(a[0], b[0]):
        assert torch.equal(x, y)
print("threads ok")
"""


def test_concurrent_first_calls_match_single_thread():
    code = _SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "threads ok" in r.stdout


def test_dropin_api_from_threads_matches_sequential():
    """render_forward / render_backward / project_scene / bin_arrays share
    the default engine; the reference's functions are pure and thread-safe
    (SURVEY.md 8(b)), so concurrent callers must each get the result a lone
    caller gets (the calls serialise on the engine's lock)."""
    import threading

    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import random_scene, random_view
    from paper_2605_18334_b200.raster import project_scene, render_backward, render_forward
    from paper_2605_18334_b200.synthetic import fp32_round

    rng = np.random.default_rng(8)
    scenes = [fp32_round(random_scene(rng, 1500 + 300 * i, sh_degree=2)) for i in range(3)]
    views = [random_view(rng, 96 + 16 * i, 64) for i in range(6)]
    jobs = [(scenes[i % 3], views[i]) for i in range(6)]
    dLs = [np.random.default_rng(10 + i).normal(size=(64, 96 + 16 * i, 3)) for i in range(6)]

    def run(i):
        sc, v = jobs[i]
        fr = render_forward(sc, v)
        g = render_backward(sc, v, fr, dLs[i])
        pr = project_scene(sc, v)
        return fr.color, fr.last_idx, g.d_mu, g.d_sh, g.g_z, pr.depth

    ref = [run(i) for i in range(6)]
    got = [None] * 6
    errs = []

    def worker(i):
        try:
            for _ in range(3):
                got[i] = run(i)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for a, b in zip(got, ref):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
