"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference package (built into oracle/_ref by
oracle/build_ref.sh from /root/reference) through its public API:
project_scene, bin_arrays, render_forward (cython backend),
_screen_gradients and render_backward.  The fixtures pin both the C oracle
(oracle/ssg_oracle.c) and the CUDA path.  Re-run after changing a case:

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from skewsplat.projection import project_scene  # noqa: E402  (reference)
from skewsplat.raster import backend as ref_backend  # noqa: E402
from skewsplat.raster.backward import _screen_gradients, render_backward  # noqa: E402
from skewsplat.raster.forward import render_forward  # noqa: E402
from skewsplat.raster.tiles import bin_arrays  # noqa: E402

from helpers import (frontal_view, random_scene, random_view, scene_arrays,  # noqa: E402
                     single_splat_scene)
from paper_2605_18334_b200.scene import Scene  # noqa: E402
from paper_2605_18334_b200.synthetic import fp32_round, frustum_scene, frustum_view  # noqa: E402


def cases():
    v = frontal_view(64, 64)
    yield "kat_single", Scene.from_primitives(
        [single_splat_scene((8.5, 8.5), v, 0.6, (1.0, 0.0, 0.0))]), v, 0.0, True
    yield "kat_pair", Scene.from_primitives(
        [single_splat_scene((8.5, 8.5), v, 0.5, (1.0, 0.0, 0.0)),
         single_splat_scene((8.5, 8.5), v, 0.5, (0.0, 0.0, 1.0))]), v, 0.0, True
    yield "kat_occluder", Scene.from_primitives(
        [single_splat_scene((32.5, 32.5), v, 0.999, (1.0, 1.0, 1.0), scale=2.0, depth=3.0),
         single_splat_scene((32.5, 32.5), v, 0.8, (0.0, 1.0, 0.0), scale=2.0, depth=8.0)]), v, 0.0, True
    for i in range(3):
        rng = np.random.default_rng(200 + i)
        sc = random_scene(rng, 12)
        yield f"skew_{i}", fp32_round(sc), random_view(rng, 48, 48), 0.3, False
    for i in range(2):
        rng = np.random.default_rng(100 + i)
        sc = random_scene(rng, 12, plain=True)
        yield f"plain_{i}", fp32_round(sc), random_view(rng, 48, 48), 0.3, False
    rng = np.random.default_rng(42)
    yield "tight_fov_33x17", fp32_round(random_scene(rng, 10)), random_view(rng, 33, 17, dist=3.0, fov_x=1.4), 0.3, False
    rng = np.random.default_rng(5)
    yield "deg0_fp64", random_scene(rng, 15, sh_degree=0), random_view(rng, 40, 40), 0.3, False
    rng = np.random.default_rng(7)
    yield "deg1_fp64", random_scene(rng, 30, sh_degree=1, skew_scale=1.5), random_view(rng, 64, 48), 0.3, False
    # strongly skewed G2-style frustum scene, scaled down
    sc = frustum_scene(n=3000, seed=3, width=160, height=96)
    yield "frustum_3k_160x96", sc, frustum_view(160, 96), 0.3, False
    rng = np.random.default_rng(11)
    yield "dense_400_96x80", fp32_round(random_scene(rng, 400, sh_degree=3, skew_scale=1.0, spread=0.8)), \
        random_view(rng, 96, 80), 0.3, False
    # skew fallback (projection.py:117-121, 133): primitives whose 3D scales
    # underflow (exp(-400)^2 = 0) have det_raw = 0 <= 1e-300, so their projected
    # skew falls back to 0 and their eta VJP is zeroed; mixed into a normal scene
    rng = np.random.default_rng(23)
    sc = fp32_round(random_scene(rng, 40, sh_degree=1, skew_scale=1.0))
    sc.log_scale[::5] = -400.0
    yield "fallback_mix", sc, random_view(rng, 56, 40), 0.3, False


def main(only=()):
    assert ref_backend.active_backend() == "cython"
    for name, scene, view, s, kat in cases():
        if only and name not in only:
            continue
        frame = render_forward(scene, view, s=s, backend_name="cython")
        proj = project_scene(scene, view, s)
        grid = bin_arrays(proj.mean2d, proj.radius, proj.depth, proj.valid, view.width, view.height)
        dL = np.random.default_rng(1).normal(size=(view.height, view.width, 3))
        _, screen = _screen_gradients(scene, view, frame, dL, backend_name="cython")
        g = render_backward(scene, view, frame, dL, backend_name="cython")
        out = dict(scene_arrays(scene))
        out.update(
            c2w=view.c2w, convention=np.array(view.convention), width=np.int64(view.width),
            height=np.int64(view.height), fov_x=np.float64(view.fov_x), s=np.float64(s),
            color=frame.color, final_T=frame.final_T, n_contrib=frame.n_contrib,
            last_idx=frame.last_idx, n_instances=np.int64(frame.n_instances),
            p_valid=proj.valid, p_mean2d=proj.mean2d, p_depth=proj.depth, p_conic=proj.conic,
            p_opair=proj.opacity_pair, p_radius=proj.radius, p_skew2d=proj.skew2d,
            p_color=proj.color, n_skew_fallback=np.int64(proj.n_skew_fallback),
            inst_prim=grid.inst_prim, inst_tile=grid.inst_tile, ranges=grid.ranges, dL=dL,
            **{f"s_{k}": v for k, v in screen.items()},
            **{f"g_{k}": getattr(g, k) for k in ("d_mu", "d_log_scale", "d_rot", "d_sh",
                                                  "d_opacity_logits", "d_beta", "d_dir",
                                                  "g_uv", "g_z")})
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(f"{name}: N={len(scene)} {view.width}x{view.height} M={frame.n_instances}")


if __name__ == "__main__":
    main(tuple(sys.argv[1:]))
