"""Per-stage device timings of one frame (CUDA events) for a synthetic config.

python tools/stage_times.py [--n 1000000] [--w 1920] [--h 1080] [--reps 5]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2605_18334_b200 import _native as N
from paper_2605_18334_b200.engine import DeviceScene, Engine, camera_struct
from paper_2605_18334_b200.synthetic import frustum_scene, frustum_view


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--w", type=int, default=1920)
    ap.add_argument("--h", type=int, default=1080)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--plain", type=float, default=0.0)
    ap.add_argument("--ball", action="store_true", help="config-4 scene (3M ball, orbit view 0, 1297x840)")
    a = ap.parse_args()
    t0 = time.time()
    if a.ball:
        from paper_2605_18334_b200.synthetic import ball_scene, orbit_views
        scene = ball_scene(3_000_000, seed=0)
        view = orbit_views(64, radius=4.0, elevation=1.2, width=1297, height=840, fov_x=0.9)[0]
        a.w, a.h = 1297, 840
    else:
        scene = frustum_scene(a.n, width=a.w, height=a.h, plain_fraction=a.plain)
        view = frustum_view(a.w, a.h)
    print(f"scene gen {time.time()-t0:.1f}s", flush=True)
    eng = Engine()
    eng.keep_inst_tile = os.environ.get("KEEP_TILE", "0") == "1"
    ds = DeviceScene.from_host(scene)
    dL = torch.from_numpy(np.random.default_rng(1).normal(size=(a.h, a.w, 3))).cuda().float()
    for rep in range(a.reps):
        eng.stage_events = {}
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        f = eng.forward(ds, view, 0.3)
        ev[1].record()
        g = eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dL, rebin=False)
        ev[2].record()
        torch.cuda.synchronize()
        print(f"rep {rep}: M={f.n_instances} fwd {ev[0].elapsed_time(ev[1]):.3f} ms "
              f"bwd {ev[1].elapsed_time(ev[2]):.3f} ms | " +
              " ".join(f"{k} {a.elapsed_time(b):.3f}" for k, v in eng.stage_events.items() for a, b in v),
              flush=True)
    print("img mean", float(f.color.mean()), "nc mean", float(f.n_contrib.float().mean()),
          "g_mu absmax", float(g.d_mu.abs().max()))


if __name__ == "__main__":
    main()
