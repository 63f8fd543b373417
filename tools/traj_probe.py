"""render_trajectory wall time (32 orbit views at 1297x840 of a 1M ball
scene) against the one-view-at-a-time loop: python tools/traj_probe.py"""

from __future__ import annotations

import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from PIL import Image  # noqa: E402

from paper_2605_18334_b200.engine import DeviceScene, default_engine  # noqa: E402
from paper_2605_18334_b200.serving import quantize_u8_device, render_trajectory  # noqa: E402
from paper_2605_18334_b200.synthetic import ball_scene, orbit_views  # noqa: E402


def main():
    scene = ball_scene(1_000_000, seed=1)
    views = orbit_views(32, radius=4.0, elevation=1.2, width=1297, height=840, fov_x=0.9)
    with tempfile.TemporaryDirectory() as d:
        render_trajectory(scene, views[:4], os.path.join(d, "w"))
        t = time.perf_counter()
        render_trajectory(scene, views, os.path.join(d, "a"))
        ta = time.perf_counter() - t
        eng = default_engine()
        t = time.perf_counter()
        ds = DeviceScene.from_host(scene, eng.device)
        os.makedirs(os.path.join(d, "b"))
        for i, v in enumerate(views):
            px = quantize_u8_device(eng.forward(ds, v, 0.3).color).cpu().numpy()
            Image.fromarray(px, mode="RGB").save(os.path.join(d, "b", f"{i:04d}.png"), format="PNG")
        tb = time.perf_counter() - t
    print(f"render_trajectory {ta * 1e3:.0f} ms, per-view loop {tb * 1e3:.0f} ms for {len(views)} views")


if __name__ == "__main__":
    main()
