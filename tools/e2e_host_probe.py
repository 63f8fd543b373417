"""Host time from entering render_forward / render_backward to the first
upload call (config 2, pinned arrays): python tools/e2e_host_probe.py"""

from __future__ import annotations

import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2605_18334_b200.raster import _link  # noqa: E402
from paper_2605_18334_b200.raster import render_backward, render_forward  # noqa: E402
from paper_2605_18334_b200.scene import Scene  # noqa: E402


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def main():
    scene, view, dL = bench.workload()
    ps = Scene(*(pinned(getattr(scene, f)) for f in Scene.ARRAY_FIELDS), background=scene.background,
               sh_degree=scene.sh_degree)
    pdL = pinned(dL)
    marks = []
    orig_up, orig_td = _link.upload_rows, _link.to_device

    def up(*a, **k):
        marks.append(("upload_rows", time.perf_counter()))
        return orig_up(*a, **k)

    def td(*a, **k):
        marks.append(("to_device", time.perf_counter()))
        return orig_td(*a, **k)
    _link.upload_rows, _link.to_device = up, td
    fwd, bwd = [], []
    for it in range(8):
        torch.cuda.synchronize()
        marks.clear()
        t0 = time.perf_counter()
        fr = render_forward(ps, view)
        f_first = marks[0][1] - t0 if marks else float("nan")
        marks.clear()
        t1 = time.perf_counter()
        render_backward(ps, view, fr, pdL)
        b_first = marks[0][1] - t1 if marks else float("nan")
        if it >= 3:
            fwd.append(f_first * 1e3)
            bwd.append(b_first * 1e3)
    print({"fwd_ms_to_first_upload": round(statistics.median(fwd), 3),
           "bwd_ms_to_first_upload": round(statistics.median(bwd), 3)})


if __name__ == "__main__":
    main()
