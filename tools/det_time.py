"""Device time of the deterministic vs the atomic backward on the config-2
frame (CUDA events, median of 5): python tools/det_time.py"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_18334_b200.engine import DeviceScene, Engine

scene, view, dL = bench.workload()
eng = Engine()
ds = DeviceScene.from_host(scene)
dLd = torch.from_numpy(dL).cuda().float()
f = eng.forward(ds, view, 0.3)
out = {}
for det in (False, True, False, True):
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dLd, rebin=False, deterministic=det)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out["det" if det else "atomic"] = round(statistics.median(ts), 3)
print(out)
