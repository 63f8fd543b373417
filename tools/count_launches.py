"""Kernels of this library launched per step (torch.profiler, CUDA
activity), for config 2's frame and config 5's pipelined training step:
python tools/count_launches.py"""

from __future__ import annotations

import collections
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2605_18334_b200.engine import DeviceScene, Engine  # noqa: E402
from paper_2605_18334_b200.synthetic import ball_scene, fp32_round, orbit_views  # noqa: E402
from paper_2605_18334_b200.train import DeviceAdam, Trainer  # noqa: E402


def ours(evs):
    c = collections.Counter()
    for e in evs:
        if e.device_type.name != "CUDA" or e.name.startswith("Memcpy") or e.name.startswith("Memset"):
            continue
        mine = any(t in e.name for t in ("ssg::", "bsort::", "osort::", "dsort::", "k_"))
        c["ours" if mine else "other"] += 1
        if not mine:
            c["other:" + e.name[:50]] += 1
    return c


def main():
    scene, view, dL = bench.workload()
    eng = Engine()
    eng.keep_inst_tile = False
    ds = DeviceScene.from_host(scene)
    dLd = torch.from_numpy(dL).cuda().float()
    for i in range(3):
        f = eng.forward(ds, view, 0.3, sync=(i == 0), defer_exact=True)
        eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dLd, rebin=False)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(4):
            f = eng.forward(ds, view, 0.3, sync=False, defer_exact=True)
            eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dLd, rebin=False)
        torch.cuda.synchronize()
    c = ours(prof.events())
    print("config 2 per frame:", {k: v / 4 for k, v in c.items()})
    sc = ball_scene(200_000, seed=1)
    views = orbit_views(4, radius=4.0, elevation=1.2, width=640, height=416, fov_x=0.9)
    teng = Engine()
    tds = DeviceScene.from_host(sc)
    targets = [teng.forward(tds, v, 0.3).color.clone() for v in views]
    start = sc.copy()
    start.mu += np.random.default_rng(5).normal(size=start.mu.shape) * 0.01
    ds2 = DeviceScene.from_host(fp32_round(start))
    tr = Trainer(teng, ds2, DeviceAdam(ds2), pipelined=True, buckets=1)
    for i in range(4):
        tr.step(views[i % 4], targets[i % 4], i)
    tr.flush()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(4, 8):
            tr.step(views[i % 4], targets[i % 4], i)
        tr.flush()
        torch.cuda.synchronize()
    c = ours(prof.events())
    print("config 5 per step:", {k: v / 4 for k, v in c.items()})


if __name__ == "__main__":
    main()
