"""Full-size parity diagnostics: the drop-in API vs the C oracle (all host
cores) on config 2 (G2: 1M skew Gaussians, 1920x1080) and config 4 view 0
(G4: 3M, 1297x840).  Prints one JSON object per config with list equality,
n_contrib / last_idx mismatch counts, pixel error histograms and gradient
error quantiles (the numbers committed under profiles/).

usage: python tools/parity_at_scale.py [c2] [c4] [--no-bwd]
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import golden_io as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2605_18334_b200.raster import render_backward, render_forward  # noqa: E402
from paper_2605_18334_b200.synthetic import ball_scene, frustum_scene, frustum_view, orbit_views  # noqa: E402

GRADS = ("d_mu", "d_log_scale", "d_rot", "d_sh", "d_opacity_logits", "d_beta", "d_dir", "g_uv", "g_z")


def _hist(d, edges=(0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 1e9)):
    h, _ = np.histogram(d, bins=np.asarray(edges, dtype=np.float64))
    return {f"<{edges[i + 1]:.0e}": int(h[i]) for i in range(len(h))}


def compare(name, scene, view, bwd=True):
    O.set_num_threads(os.cpu_count() or 1)
    out = {"config": name, "n": int(scene.mu.shape[0]), "width": view.width, "height": view.height,
           "oracle_threads": O.num_threads()}
    t0 = time.time()
    fr = render_forward(scene, view)
    out["gpu_fwd_s"] = round(time.time() - t0, 2)
    from paper_2605_18334_b200.engine import default_engine
    out["exact_path_pixels"] = default_engine().redo_pixels()
    t0 = time.time()
    ref = O.render_forward(scene, view)
    out["oracle_fwd_s"] = round(time.time() - t0, 2)
    out["M"] = [fr.n_instances, ref.n_instances]
    d = np.abs(fr.color - ref.color).max(axis=2)
    out["pixel_max_abs"] = float(d.max())
    out["pixel_hist"] = _hist(d.ravel())
    out["final_T_max_abs"] = float(np.abs(fr.final_T - ref.final_T).max())
    out["n_contrib_mismatch"] = int(np.sum(fr.n_contrib != ref.n_contrib))
    out["last_idx_mismatch"] = int(np.sum(fr.last_idx != ref.last_idx))
    if bwd:
        dL = np.random.default_rng(1).normal(size=(view.height, view.width, 3))
        t0 = time.time()
        g = render_backward(scene, view, fr, dL)
        out["gpu_bwd_s"] = round(time.time() - t0, 2)
        t0 = time.time()
        rg = O.render_backward(scene, view, ref, dL)
        out["oracle_bwd_s"] = round(time.time() - t0, 2)
        ge = {}
        for k in GRADS:
            e = G.rel_floor(getattr(g, k), getattr(rg, k)).ravel()
            ge[k] = {"frac_le_1e-3": float(np.mean(e <= 1e-3)), "p999": float(np.quantile(e, 0.999)),
                     "max": float(e.max())}
        out["grad_rel_floor"] = ge
    return out


def main():
    args = sys.argv[1:] or ["c2"]
    bwd = "--no-bwd" not in args
    res = []
    if "c2" in args:
        res.append(compare("config2_G2", frustum_scene(1_000_000, seed=0), frustum_view(), bwd))
        print(json.dumps(res[-1]), flush=True)
    if "c4" in args:
        view = orbit_views(64, radius=4.0, elevation=1.2, width=1297, height=840, fov_x=0.9)[0]
        res.append(compare("config4_G4_view0", ball_scene(3_000_000, seed=0), view, bwd))
        print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__":
    main()
