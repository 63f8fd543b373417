"""How much of a config-5 training step is the per-step host read-back?
Times training_step as shipped against the same GPU work with the read-back
removed (instance-count check and finite-loss branch skipped) -- a probe,
not a valid training loop."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2605_18334_b200 import _native as N
from paper_2605_18334_b200.engine import DeviceScene, Engine
from paper_2605_18334_b200.synthetic import ball_scene, fp32_round, orbit_views
from paper_2605_18334_b200.train import DeviceAdam, Trainer, training_step, _stream


def main():
    views = orbit_views(64, radius=4.0, elevation=1.2, width=1297, height=840, fov_x=0.9)
    scene = ball_scene(2_000_000, seed=0)
    eng = Engine()
    eng.keep_inst_tile = False
    tgt_ds = DeviceScene.from_host(scene)
    targets = torch.empty((8, 840, 1297, 3), dtype=torch.float32, device="cuda")
    for i in range(8):
        eng.forward(tgt_ds, views[i], 0.3, color_out=targets[i])
    del tgt_ds
    start = scene.copy()
    start.mu += np.random.default_rng(5).normal(size=start.mu.shape) * 0.01
    ds = DeviceScene.from_host(fp32_round(start))
    adam = DeviceAdam(ds)
    tr = Trainer(eng, ds, adam)

    def shipped(i):
        training_step(eng, ds, adam, views[i % 8], targets[i % 8])

    def nosync(i):
        view, target = views[i % 8], targets[i % 8]
        f = eng.forward(ds, view, 0.3, sync=False)
        lossfn = tr.loss_for(f.width, f.height)
        dL = lossfn(f.color, target)
        n = ds.n
        if tr.d_beta is None:
            tr.d_beta = torch.empty((n, 3), dtype=torch.float32, device=eng.device)
        lossfn.sums[2].zero_()
        g = eng.backward(ds, view, 0.3, f.final_T, f.last_idx, dL, rebin=False)
        N.check(N.lib().ssg_regularize(n, ds.beta.data_ptr(), ds.opacity_logits.data_ptr(), g.d_eta.data_ptr(),
                                       tr.cfg.lambda_beta_reg, tr.cfg.lambda_opacity_reg, tr.d_beta.data_ptr(),
                                       g.d_opacity_logits.data_ptr(), lossfn.sums.data_ptr(),
                                       _stream(eng.device)), "ssg_regularize")
        adam.step(g, i, d_beta=tr.d_beta[:n])

    for fn, name in ((shipped, "shipped"), (nosync, "no read-back"), (shipped, "shipped")):
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(20):
            fn(i)
        b.record()
        torch.cuda.synchronize()
        print(f"{name}: {a.elapsed_time(b) / 20:.3f} ms/step")
    eng.instances()


if __name__ == "__main__":
    main()
