"""View-parallel training step (config 5) on top of the rasterizer.

One process per GPU.  Every rank holds the full scene and optimizer state
(replicated); per step each rank renders its own training view(s) forward +
backward, the packed per-Gaussian gradient buffer is SUM all-reduced and
g_z is MAX all-reduced over NCCL, and every rank applies
the identical Adam step (optimize/adam.py:71-97, ssg_adam_step), so the
replicas stay bit-identical.  The reference trains one view per step
(trainer.py:127-129); with R ranks a step here consumes R views, so it is
checked at gradient level: the reduced gradients equal the sum of per-view
gradients.

The photometric loss is L1 (the L1 part of losses.py:139-149; SSIM and the
regularizers are outside the hot-path scope).
"""

from __future__ import annotations

import ctypes
import dataclasses

import torch
import torch.distributed as dist

from . import _native as N
from .engine import DeviceGrads, DeviceScene, Engine

SUM_FIELDS = ("d_mu", "d_log_scale", "d_rot", "d_sh", "d_opacity_logits", "d_eta", "g_uv")


@dataclasses.dataclass
class LearningRates:
    """optimize/config.py:19-25 defaults; lr_beta drives beta and dir."""
    mu: float = 1e-3
    log_scale: float = 5e-3
    rot: float = 2e-3
    sh: float = 2.5e-3
    opacity: float = 2.5e-2
    beta: float = 1e-4


def allreduce_gradients(grads: DeviceGrads, group=None) -> None:
    """SUM of the packed gradient buffer, MAX of g_z (one call each)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dist.all_reduce(grads.flat, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(grads.g_z, op=dist.ReduceOp.MAX, group=group)


def l1_loss_grad(color: torch.Tensor, target: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """mean |c - t| and its pixel gradient sign(c - t) / (3P)."""
    diff = color - target
    return diff.abs().mean(), torch.sign(diff) / diff.numel()


class DeviceAdam:
    """Adam state on the device (fp32 moments) bound to a DeviceScene."""

    def __init__(self, ds: DeviceScene, lr: LearningRates | None = None):
        self.ds = ds
        self.lr = lr or LearningRates()
        self.t = 0
        dev = ds.mu.device
        z = lambda *shape: torch.zeros(shape, dtype=torch.float32, device=dev)  # noqa: E731
        n, K = ds.n, ds.K
        self.m = {"mu": z(n, 3), "log_scale": z(n, 3), "rot": z(n, 4), "sh": z(n, K, 3), "logits": z(n, 2),
                  "eta": z(n, 3)}
        self.v = {k: torch.zeros_like(v) for k, v in self.m.items()}
        self.row_ok = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        self.n_skipped_dev = torch.zeros(1, dtype=torch.int32, device=dev)

    def step(self, grads: DeviceGrads) -> None:
        ds = self.ds
        self.t += 1
        p = N.SsgParams()
        p.n, p.sh_degree, p.sh_coeffs = ds.n, ds.sh_degree, ds.K
        p.mu, p.log_scale, p.rot = ds.mu.data_ptr(), ds.log_scale.data_ptr(), ds.rot.data_ptr()
        p.sh, p.opacity_logits = ds.sh.data_ptr(), ds.opacity_logits.data_ptr()
        p.beta, p.dir = ds.beta.data_ptr(), ds.dir.data_ptr()
        g = N.SsgGradBuffers()
        g.d_mu, g.d_log_scale, g.d_rot = grads.d_mu.data_ptr(), grads.d_log_scale.data_ptr(), grads.d_rot.data_ptr()
        g.d_sh, g.d_opacity_logits = grads.d_sh.data_ptr(), grads.d_opacity_logits.data_ptr()
        g.d_eta = grads.d_eta.data_ptr()
        s = N.SsgAdamState()
        for f, key in (("mu", "mu"), ("log_scale", "log_scale"), ("rot", "rot"), ("sh", "sh"),
                       ("logits", "logits"), ("eta", "eta")):
            setattr(s, "m_" + f, self.m[key].data_ptr())
            setattr(s, "v_" + f, self.v[key].data_ptr())
        s.row_ok, s.n_skipped = self.row_ok.data_ptr(), self.n_skipped_dev.data_ptr()
        hp = N.SsgAdamHparams()
        hp.t = self.t
        hp.lr_mu, hp.lr_scale, hp.lr_rot = self.lr.mu, self.lr.log_scale, self.lr.rot
        hp.lr_sh, hp.lr_opacity, hp.lr_beta = self.lr.sh, self.lr.opacity, self.lr.beta
        N.check(N.lib().ssg_adam_step(ctypes.byref(p), ctypes.byref(g), ctypes.byref(s), ctypes.byref(hp),
                                      torch.cuda.current_stream(ds.mu.device).cuda_stream), "ssg_adam_step")

    def n_skipped(self) -> int:
        return int(self.n_skipped_dev.item())


def training_step(eng: Engine, ds: DeviceScene, adam: DeviceAdam, view, target: torch.Tensor,
                  s: float = 0.3, group=None) -> torch.Tensor:
    """One view-parallel step: render this rank's view, L1 loss, backward,
    all-reduce gradients, Adam.  Returns the (device) loss of this rank."""
    f = eng.forward(ds, view, s)
    loss, dL = l1_loss_grad(f.color, target)
    grads = eng.backward(ds, view, s, f.final_T, f.last_idx, dL.contiguous(), rebin=False)
    allreduce_gradients(grads, group)
    adam.step(grads)
    return loss
