"""Visit counts of the backward under coarser warp blocks, from the forward's
blend masks (config 2): (8x8 block, instance) visits as shipped vs the union of
vertically / horizontally adjacent blocks (an 8x16 / 16x8 block per warp)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2605_18334_b200.engine import DeviceScene, Engine

scene, view, dL = bench.workload()
eng = Engine()
ds = DeviceScene.from_host(scene)
f = eng.forward(ds, view, 0.3)
m = eng.last_m
words = eng.blend_mask.cpu().numpy().view(np.uint32)
rg = eng.ranges.cpu().numpy()
pc = np.vectorize(lambda x: bin(int(x)).count("1"))
v88 = v816 = v168 = 0
for t in range(rg.shape[0]):
    s, e = rg[t]
    if e <= s: continue
    nch = (e - s + 31) // 32
    base = (s // 32 + t)
    w = words[(base + np.arange(nch))[:, None] * 4 + np.arange(4)[None, :]]  # (chunk, warp)
    v88 += int(np.unpackbits(w.view(np.uint8)).sum())
    v816 += int(np.unpackbits((w[:, 0] | w[:, 2]).view(np.uint8)).sum() + np.unpackbits((w[:, 1] | w[:, 3]).view(np.uint8)).sum())
    v168 += int(np.unpackbits((w[:, 0] | w[:, 1]).view(np.uint8)).sum() + np.unpackbits((w[:, 2] | w[:, 3]).view(np.uint8)).sum())
print({"visits_8x8": v88, "visits_8x16": v816, "visits_16x8": v168, "ratio_8x16": v816 / v88, "ratio_16x8": v168 / v88})
