"""Config-2 frames (fwd + bwd) with k engines in flight on their own streams,
each frame a CUDA graph: throughput of independent frames (a serving data
point; bench.py's headline times one frame at a time).
python tools/c2_lanes.py [k ...]"""

from __future__ import annotations

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2605_18334_b200.engine import DeviceScene, Engine  # noqa: E402


def main():
    scene, view, dL = bench.workload()
    ds = DeviceScene.from_host(scene)
    dLd = torch.from_numpy(dL).cuda().float()
    for k in [int(x) for x in sys.argv[1:]] or [1, 2, 3]:
        engines = [Engine() for _ in range(k)]
        graphs, streams = [], []
        for eng in engines:
            eng.keep_inst_tile = False

            def step(eng=eng, sync=False):
                f = eng.forward(ds, view, 0.3, sync=sync, defer_exact=True)
                eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dLd, rebin=False)
            for i in range(3):
                step(sync=(i == 0))
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            graphs.append(g)
            streams.append(torch.cuda.Stream())
        steps = 60
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for st in streams:
                st.wait_event(e0)
            for i in range(steps):
                j = i % k
                with torch.cuda.stream(streams[j]):
                    graphs[j].replay()
            for st in streams:
                ev = torch.cuda.Event()
                ev.record(st)
                torch.cuda.current_stream().wait_event(ev)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        for eng in engines:
            eng.instances()
        print(f"lanes {k}: {ms:.3f} ms per frame, {1000 / ms:.1f} views/s")


if __name__ == "__main__":
    main()
