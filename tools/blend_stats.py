"""Blend event counters on config 2 (diagnostic build).

python -m paper_2605_18334_b200.build --stats
SSG_B200_LIB=paper_2605_18334_b200/libssg_b200_stats.so python tools/blend_stats.py
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2605_18334_b200 import _native as N
from paper_2605_18334_b200.engine import DeviceScene, Engine
from paper_2605_18334_b200.synthetic import frustum_scene, frustum_view

NAMES = {0: "fwd hits (warp x instance, exact ellipse test)", 1: "fwd hits with a blending pixel",
         2: "fwd sum over batches of the slowest warp's hits", 3: "fwd sum over batches of all warps' hits",
         4: "fwd sum over tiles of the slowest warp's hits", 5: "fwd sum over tiles of all warps' hits",
         16: "bwd visited (warp x instance)", 17: "bwd visited with a contributing pixel",
         18: "bwd contributing pixels"}


def main():
    L = N.lib()
    L.ssg_test_blend_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
    plain = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
    scene = frustum_scene(1_000_000, width=1920, height=1080, plain_fraction=plain)
    view = frustum_view(1920, 1080)
    eng = Engine()
    ds = DeviceScene.from_host(scene)
    dL = torch.from_numpy(np.random.default_rng(1).normal(size=(1080, 1920, 3))).cuda().float()
    buf = (ctypes.c_ulonglong * 32)()
    f = eng.forward(ds, view, 0.3)
    eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dL, rebin=False)
    torch.cuda.synchronize()
    L.ssg_test_blend_stats(buf, 1)
    for i, name in NAMES.items():
        print(f"{i:3d} {name:45s} {buf[i]:>16,d}")
    print("M", f.n_instances)
    if buf[3]:
        print(f"fwd barrier imbalance: 8 x max / total = {8 * buf[2] / buf[3]:.3f} per batch, "
              f"{8 * buf[4] / max(buf[5], 1):.3f} per tile (1 = balanced)")


if __name__ == "__main__":
    main()
