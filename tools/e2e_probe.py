"""Where does an end-to-end config-2 frame (render_forward + render_backward
on pinned fp64 host arrays) spend its time?  Host wall clock per phase,
with a device synchronise after each so the phases do not overlap."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2605_18334_b200.camera import to_opencv
from paper_2605_18334_b200.engine import DeviceScene, default_engine
from paper_2605_18334_b200.raster import render_backward, render_forward
from paper_2605_18334_b200.raster.forward import frame_to_host
from paper_2605_18334_b200.scene import Scene
from paper_2605_18334_b200.synthetic import frustum_scene, frustum_view


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def main():
    scene = frustum_scene(1_000_000)
    view = frustum_view()
    ps = Scene(*(pinned(getattr(scene, f)) for f in Scene.ARRAY_FIELDS), background=scene.background,
               sh_degree=scene.sh_degree)
    dL = pinned(np.random.default_rng(1).normal(size=(1080, 1920, 3)))
    fr = render_forward(ps, view)
    render_backward(ps, view, fr, dL)
    torch.cuda.synchronize()
    eng = default_engine()
    ov = to_opencv(view)
    for rep in range(3):
        t = [time.perf_counter()]
        ds = DeviceScene.from_host(ps, eng.device)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        f = eng.forward(ds, ov, 0.3)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        fr = frame_to_host(f)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        g = render_backward(ps, view, fr, dL)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        ms = np.diff(t) * 1e3
        print(f"upload {ms[0]:.2f}  forward {ms[1]:.2f}  frame->host {ms[2]:.2f}  render_backward {ms[3]:.2f}  "
              f"total {sum(ms):.2f} ms")
    t0 = time.perf_counter()
    for _ in range(3):
        fr = render_forward(ps, view)
        g = render_backward(ps, view, fr, dL)
    torch.cuda.synchronize()
    print(f"API e2e {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms/frame")


if __name__ == "__main__":
    main()
