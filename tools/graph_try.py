"""Capture one config-2 frame (forward + backward) in a CUDA graph and
compare replay with eager launches: outputs and time per frame."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2605_18334_b200.engine import DeviceScene, Engine
from paper_2605_18334_b200.synthetic import frustum_scene, frustum_view


def main():
    scene = frustum_scene(1_000_000)
    view = frustum_view()
    eng = Engine()
    eng.keep_inst_tile = False
    ds = DeviceScene.from_host(scene)
    dL = torch.from_numpy(np.random.default_rng(1).normal(size=(1080, 1920, 3))).cuda().float()

    def step(sync=False):
        f = eng.forward(ds, view, 0.3, sync=sync)
        return f, eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dL, rebin=False)

    for i in range(4):
        f, g = step(sync=(i == 0))
    torch.cuda.synchronize()
    ref_color = f.color.clone()
    ref_mu = g.d_mu.clone()

    def timeit(fn, k=30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        a.record()
        for _ in range(k):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / k

    t_eager = timeit(lambda: step())
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()  # warm on the capture stream
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    with torch.cuda.graph(graph):
        f2, g2 = step()
    graph.replay()
    torch.cuda.synchronize()
    print("color equal:", torch.equal(f2.color, ref_color), "d_mu maxdiff:",
          float((g2.d_mu - ref_mu).abs().max()), "M:", eng.instances())
    t_graph = timeit(lambda: graph.replay())
    print(f"eager {t_eager:.4f} ms/frame, graph {t_graph:.4f} ms/frame")


if __name__ == "__main__":
    main()
