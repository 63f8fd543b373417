"""Timeline of one drop-in render_forward + render_backward (config 2,
pinned host arrays) from torch.profiler: copies and kernels per stream, ms
from the first event: python tools/e2e_trace.py [forward|backward]"""

from __future__ import annotations

import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

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
    scene, view, dL = bench.workload()
    if os.environ.get("PAGEABLE"):  # the caller's own numpy arrays
        ps, pdL = scene, dL
    else:
        ps = Scene(*(pinned(getattr(scene, f)) for f in Scene.ARRAY_FIELDS), background=scene.background,
                   sh_degree=scene.sh_degree)
        pdL = pinned(dL)
    for _ in range(3):
        fr = render_forward(ps, view)
        render_backward(ps, view, fr, pdL)
    which = sys.argv[1] if len(sys.argv) > 1 else "backward"
    fr = render_forward(ps, view)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        if which == "forward":
            render_forward(ps, view)
        else:
            render_backward(ps, view, fr, pdL)
        torch.cuda.synchronize()
    print(f"== render_{which}")
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    cpu = [e for e in prof.events() if e.device_type.name == "CPU" and e.name in ("render_backward",)]
    t0 = min(e.time_range.start for e in evs)
    rows = []
    for e in evs:
        rows.append((e.time_range.start - t0, e.time_range.end - t0, getattr(e, "device_resource_id", -1), e.name[:60]))
    rows.sort()
    # merge: per stream, print spans
    for st in sorted({r[2] for r in rows}):
        rs = [r for r in rows if r[2] == st]
        print(f"stream {st}: {len(rs)} events, {rs[0][0]/1e3:.2f}-{max(r[1] for r in rs)/1e3:.2f} ms, busy "
              f"{sum(r[1]-r[0] for r in rs)/1e3:.2f} ms")
        for r in rs:
            if r[1] - r[0] > 150:
                print(f"   {r[0]/1e3:7.2f} {r[1]/1e3:7.2f}  {r[3]}")
    ct = [e for e in prof.events() if e.device_type.name == "CPU"]
    c0 = min(e.time_range.start for e in ct)
    print("cpu span ms", (max(e.time_range.end for e in ct) - c0) / 1e3, "gpu first event after cpu start ms",
          (t0 - c0) / 1e3)


if __name__ == "__main__":
    main()
