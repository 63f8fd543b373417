"""Host-clock breakdown of the drop-in e2e frame (render_forward +
render_backward on the config-2 scene with pinned host arrays):
python tools/e2e_phases.py  -> one JSON line of per-phase ms (median of 5)."""

from __future__ import annotations

import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2605_18334_b200.engine import DeviceScene, camera_struct, default_engine  # noqa: E402
from paper_2605_18334_b200.raster import forward as F  # noqa: E402
from paper_2605_18334_b200.raster import backward as B  # noqa: E402
from paper_2605_18334_b200.camera import to_opencv  # noqa: E402
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
    view = to_opencv(view)
    eng = default_engine()
    phases = {}

    def tick(name, t0):
        torch.cuda.synchronize()
        t = time.perf_counter()
        phases.setdefault(name, []).append((t - t0) * 1e3)
        return t

    for it in range(7):
        torch.cuda.synchronize()
        t = t_all = time.perf_counter()
        ds = DeviceScene.from_host(ps, eng.device)
        t = tick("fwd_upload", t)
        f = eng.forward(ds, view, 0.3)
        t = tick("fwd_device", t)
        fr = F.frame_to_host(f)
        t = tick("fwd_download", t)
        dl = B._validate(ps, view, fr, pdL)
        t = tick("bwd_validate", t)
        e, g = B._device_backward(ps, view, fr, dl)
        t = tick("bwd_upload+device", t)
        outs = [B._host(x) for x in (g.d_mu, g.d_log_scale, g.d_rot, g.d_sh, g.d_opacity_logits,
                                     g.d_eta, g.d_eta, g.g_uv, g.g_z)]
        t = tick("bwd_download", t)
        del outs, fr
        tick("total", t_all)
        if it == 1:
            phases.clear()
    # the upload alone, and the backward device part alone
    for _ in range(5):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ds2 = DeviceScene.from_host(ps, eng.device)
        t = tick("upload_only", t)
        m = eng.project_and_bin(ds2, camera_struct(view, 0.3))
        t = tick("project_and_bin", t)
        ft = torch.from_numpy(np.ascontiguousarray(fr_T := F.frame_to_host(eng.forward(ds2, view, 0.3)).final_T))
        t = time.perf_counter()
        g = eng.backward(ds2, view, 0.3, ft.cuda().float(), eng.forward(ds2, view, 0.3).last_idx,
                         torch.from_numpy(dL).cuda().float(), rebin=False, deterministic=True)
        tick("fwd+bwd_det_device", t)
    out = {k: round(statistics.median(v), 3) for k, v in phases.items()}
    # the public calls as bench.py times them (previous bundles alive / dropped)
    from paper_2605_18334_b200.raster import render_backward, render_forward
    for keep in (True, False):
        ts = []
        fr = g = None
        for _ in range(6):
            if not keep:
                fr = g = None
            torch.cuda.synchronize()
            t = time.perf_counter()
            fr = render_forward(ps, view)
            g = render_backward(ps, view, fr, pdL)
            torch.cuda.synchronize()
            ts.append(round((time.perf_counter() - t) * 1e3, 2))
        out["api_keep" if keep else "api_drop"] = ts
    print(json.dumps(out))


if __name__ == "__main__":
    main()
