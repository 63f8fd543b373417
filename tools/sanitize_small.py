"""A small forward + backward through every blend mode, for compute-sanitizer
(memcheck / racecheck / synccheck): python tools/sanitize_small.py

Covers the fp32 kernels, the exact path (all_exact), the deterministic
backward, the plugin slot's per-instance slots, both depth sorts (the
cooperative one below 2M keys via the binning, the onesweep one through the
sort hook) and the counting scatter; the view-batched projection with its
lanes (priority streams), the pipelined + bucketed training step (step-value
kernel, range-wise projection backward / Adam) and the deterministic
backward's half batches; the drop-in render_forward / render_backward
(speculative forward on the kept scene, chunked backward)."""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import random_scene, random_view  # noqa: E402
from paper_2605_18334_b200 import _native as N  # noqa: E402
from paper_2605_18334_b200 import plugin  # noqa: E402
from paper_2605_18334_b200.engine import DeviceScene, Engine  # noqa: E402
from paper_2605_18334_b200.synthetic import fp32_round  # noqa: E402


def main():
    rng = np.random.default_rng(3)
    scene = fp32_round(random_scene(rng, 300, sh_degree=2))
    view = random_view(rng, 72, 40)
    eng = Engine()
    ds = DeviceScene.from_host(scene)
    dL = torch.from_numpy(np.random.default_rng(4).normal(size=(40, 72, 3))).float().cuda()
    for all_exact in (False, True):
        eng.all_exact = all_exact
        f = eng.forward(ds, view, 0.3)
        eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dL, rebin=False)
        eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dL, rebin=False, deterministic=True)
        f = eng.forward(ds, view, 0.3, defer_exact=True)
        eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dL, rebin=False)
    torch.cuda.synchronize()
    # plugin slot (per-instance slots)
    from oracle import oracle as O
    proj = O.project(scene, view, 0.3)
    grid = O.bin_arrays(proj.mean2d, proj.radius, proj.depth, proj.valid, 72, 40)
    img, T, nc, li = plugin.forward_tiles(proj.mean2d, proj.conic, proj.skew2d, proj.opacity_pair, proj.color,
                                          grid.inst_prim, grid.ranges, grid.tiles_x, 72, 40, scene.background)
    plugin.backward_tiles(proj.mean2d, proj.conic, proj.skew2d, proj.opacity_pair, proj.color, grid.inst_prim,
                          grid.ranges, grid.tiles_x, 72, 40, scene.background, T, li,
                          np.random.default_rng(5).normal(size=(40, 72, 3)))
    # onesweep sort through the hook (>= 2M keys)
    L = N.lib()
    n = 2_100_000
    keys = torch.from_numpy(np.random.default_rng(6).uniform(2, 12, n).view(np.int64)).cuda()
    vals = torch.empty(n, dtype=torch.int32, device="cuda")
    tmp = torch.empty(int(L.ssg_test_sort_temp_bytes(n, 8)), dtype=torch.uint8, device="cuda")
    N.check(L.ssg_test_sort(keys.data_ptr(), vals.data_ptr(), 8, 1, n, 8, tmp.data_ptr(),
                            torch.cuda.current_stream().cuda_stream), "sort")
    torch.cuda.synchronize()
    # view batches (ssg_preprocess_forward_views, 2 lanes, 11 views: 8 + 3)
    from paper_2605_18334_b200.views import render_views
    views = [random_view(rng, 72, 40) for _ in range(11)]
    render_views(ds, views, engine=[Engine(), Engine()])
    # a pipelined, bucketed training step (ssg_step_value, range-wise
    # projection backward, regularizer and Adam)
    from paper_2605_18334_b200.train import DeviceAdam, IntervalStats, Trainer
    tds = DeviceScene.from_host(scene)
    teng = Engine()
    teng.deterministic = True
    tr = Trainer(teng, tds, DeviceAdam(tds), pipelined=True, buckets=3)
    stats = IntervalStats(tds.n, teng.device)
    target = torch.rand((40, 72, 3), device="cuda")
    for it in range(3):
        tr.step(views[it], target, it, stats=stats)
    tr.flush()
    torch.cuda.synchronize()
    # the drop-in calls: speculative forward (kept scene), chunked backward
    # (row-range projection backward, two copy streams), a changed scene
    from paper_2605_18334_b200.raster import render_backward, render_forward
    dLh = np.random.default_rng(7).normal(size=(40, 72, 3))
    for sc in (scene, scene, scene.copy()):
        fr = render_forward(sc, view)
        render_backward(sc, view, fr, dLh)
    moved = scene.copy()
    moved.sh[-1, 0, 0] += 0.5
    fr = render_forward(moved, view)
    render_backward(moved, view, fr, dLh)
    torch.cuda.synchronize()
    print("sanitize_small: ok")


if __name__ == "__main__":
    main()
