"""Host-clock split of the drop-in e2e frame into render_forward and
render_backward (config-2 scene, pinned host arrays), and the two link
directions alone: python tools/e2e_split.py -> one JSON line (ms, medians)."""

from __future__ import annotations

import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2605_18334_b200.raster import render_backward, render_forward  # noqa: E402
from paper_2605_18334_b200.scene import Scene  # noqa: E402


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def main():
    from paper_2605_18334_b200.raster import backward as RB
    if len(sys.argv) > 1:
        RB._PIPE_CHUNKS = int(sys.argv[1])

    scene, view, dL = bench.workload()
    if os.environ.get("PAGEABLE"):  # the caller's own numpy arrays, as a reference user passes them
        ps, pdL = scene, dL
    else:
        ps = Scene(*(pinned(getattr(scene, f)) for f in Scene.ARRAY_FIELDS), background=scene.background,
                   sh_degree=scene.sh_degree)
        pdL = pinned(dL)
    res = {"fwd": [], "bwd": [], "h2d_528MB": [], "d2h_528MB": [], "both_528MB": []}
    for it in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fr = render_forward(ps, view)
        t1 = time.perf_counter()
        g = render_backward(ps, view, fr, pdL)
        t2 = time.perf_counter()
        del g
        if it >= 3:
            res["fwd"].append((t1 - t0) * 1e3)
            res["bwd"].append((t2 - t1) * 1e3)
    hb = torch.empty(66_000_000, dtype=torch.float64, pin_memory=True)
    hb2 = torch.empty_like(hb, pin_memory=True)
    db = torch.empty(hb.shape, dtype=torch.float64, device="cuda")
    db2 = torch.empty_like(db)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for it in range(5):
        torch.cuda.synchronize()
        t = time.perf_counter()
        db.copy_(hb, non_blocking=True)
        torch.cuda.synchronize()
        res["h2d_528MB"].append((time.perf_counter() - t) * 1e3)
        t = time.perf_counter()
        hb2.copy_(db2, non_blocking=True)
        torch.cuda.synchronize()
        res["d2h_528MB"].append((time.perf_counter() - t) * 1e3)
        t = time.perf_counter()
        with torch.cuda.stream(s1):
            db.copy_(hb, non_blocking=True)
        with torch.cuda.stream(s2):
            hb2.copy_(db2, non_blocking=True)
        torch.cuda.synchronize()
        res["both_528MB"].append((time.perf_counter() - t) * 1e3)
    print(json.dumps({k: round(statistics.median(v), 3) for k, v in res.items()}))


if __name__ == "__main__":
    main()
