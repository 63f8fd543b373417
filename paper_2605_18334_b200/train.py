"""View-parallel training step (config 5) on top of the rasterizer.

Mirrors the reference's training glue on the device:
  TrainConfig            optimize/config.py:9-61 (fields, defaults, validate,
                         position_lr_at)
  image_loss             optimize/losses.py:103-113 ((1-l) L1 + l (1 - SSIM),
                         analytic pixel gradient; ssg_image_loss)
  regularizers           optimize/losses.py:116-136 (ssg_regularize)
  DeviceAdam             optimize/adam.py:53-97 (ssg_adam_step: skip non-finite
                         rows, bias-corrected moments, per-field rates, quaternion
                         renormalisation; beta and dir keep separate moments)
  IntervalStats          trainer.py:40-58 (ssg_interval_stats_add)
  training_step          fit2d.py:62-78 (render, loss, stop on a non-finite loss,
                         backward, stats before the regularizers, Adam)

One process per GPU.  Every rank holds the full scene and optimizer state
(replicated); per step each rank renders its own training view forward +
backward, the packed per-Gaussian gradient buffer is SUM all-reduced and g_z
is MAX all-reduced over NCCL, and every rank applies the
identical regularizers and Adam step, so the replicas stay bit-identical.
The reference trains one view per step (trainer.py:127-129); with R ranks a
step consumes R views, so it is checked at gradient level: the reduced
gradients equal the sum of per-view gradients.
"""

from __future__ import annotations

import ctypes
import dataclasses
import math

import torch
import torch.distributed as dist

from . import _native as N
from .engine import DeviceGrads, DeviceScene, Engine, camera_struct

SUM_FIELDS = ("d_mu", "d_log_scale", "d_rot", "d_sh", "d_opacity_logits", "d_eta", "g_uv")


@dataclasses.dataclass
class TrainConfig:
    """optimize/config.py:9-38 (same fields and defaults)."""
    lr_position: float = 1e-3
    lr_position_final: float | None = None
    lr_scale: float = 5e-3
    lr_rot: float = 2e-3
    lr_opacity: float = 2.5e-2
    lr_sh: float = 2.5e-3
    lr_beta: float = 1e-4
    tau_uv: float = 1e-3
    tau_z: float = math.nan
    densify_interval: int = 100
    densify_start: int = 500
    densify_end: int = 15000
    prune_alpha: float = 5e-3
    split_scale_threshold: float = 0.05
    max_screen_radius: float | None = None
    lambda_ssim: float = 0.2
    lambda_beta_reg: float = 1e-4
    lambda_opacity_reg: float = 1e-3
    iterations: int = 3000
    seed: int = 0

    def validate(self):
        """config.py:40-55."""
        for name in ("lr_position", "lr_scale", "lr_rot", "lr_opacity", "lr_sh"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be > 0")
        for name in ("lr_beta", "tau_uv", "prune_alpha", "split_scale_threshold",
                     "lambda_ssim", "lambda_beta_reg", "lambda_opacity_reg"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")
        if not (math.isnan(self.tau_z) or self.tau_z >= 0):
            raise ValueError("tau_z must be >= 0, nan (auto), or inf")
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")
        return self

    def position_lr_at(self, iteration: int) -> float:
        """config.py:57-61: optional exponential decay of the position rate."""
        if self.lr_position_final is None:
            return self.lr_position
        t = min(max(iteration / max(self.iterations, 1), 0.0), 1.0)
        return self.lr_position * (self.lr_position_final / self.lr_position) ** t


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _world(group=None) -> int:
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def any_rank(flag: bool, group=None, device=None) -> bool:
    """True on every rank when `flag` is true on any rank (MAX all-reduce)."""
    if _world(group) == 1:
        return bool(flag)
    t = torch.tensor([1.0 if flag else 0.0], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return bool(t.item() > 0)


def allreduce_gradients(grads: DeviceGrads, group=None) -> None:
    """SUM of the packed gradient buffer, MAX of g_z (one call each)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dist.all_reduce(grads.flat, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(grads.g_z, op=dist.ReduceOp.MAX, group=group)


def bucket_bounds(n: int, buckets: int, align: int = 128) -> list:
    """[a, b) primitive ranges covering [0, n): `buckets` near-equal parts
    with inner bounds on `align` multiples (keeps every field row of a
    range 16-byte aligned and K8's 128-primitive warp groups whole)."""
    buckets = max(1, int(buckets))
    cuts = [0]
    for i in range(1, buckets):
        c = (n * i // buckets) // align * align
        if c > cuts[-1]:
            cuts.append(c)
    if n > cuts[-1] or not n:
        cuts.append(n)
    return [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]


def bucketed_allreduce(grads: DeviceGrads, bounds: list, group=None, produce=None, consume=None,
                       comm_stream=None) -> None:
    """Per primitive range [a, b) of `bounds`, in order: produce(a, b)
    writes the range's gradients (compute stream), one grouped SUM
    all-reduce of the range's rows of every SUM field (DeviceGrads.
    SUM_FIELDS) plus a MAX all-reduce of its g_z rows runs on
    `comm_stream`, then consume(a, b) uses the reduced rows (compute stream).
    On CUDA every produce is queued first, so range i's all-reduce overlaps
    the production of the later ranges, and consume(i) overlaps the
    all-reduce of range i + 1 (the streams are ordered by events; NCCL's
    own stream waits for the issuing stream).  Without a comm stream (CPU /
    gloo, or one process) the same calls run in program order.  The result
    equals allreduce_gradients + one consume over everything: the reduced
    values of a row do not depend on how rows are grouped."""
    world = _world(group)
    cuda = comm_stream is not None and grads.g_z.is_cuda
    nccl = world > 1 and dist.get_backend(group) == "nccl"

    def reduce_range(a, b):
        if world == 1:
            return
        g = grads.rows(a, b)
        if cuda and not nccl:  # gloo over CUDA tensors: no coalescing support
            for f in DeviceGrads.SUM_FIELDS:
                dist.all_reduce(getattr(g, f), op=dist.ReduceOp.SUM, group=group)
        else:
            with dist._coalescing_manager(group, grads.g_z.device if cuda else None, async_ops=True) as cm:
                for f in DeviceGrads.SUM_FIELDS:
                    dist.all_reduce(getattr(g, f), op=dist.ReduceOp.SUM, group=group)
            cm.wait()
        dist.all_reduce(g.g_z, op=dist.ReduceOp.MAX, group=group)

    if not cuda:
        for a, b in bounds:
            if produce:
                produce(a, b)
        for a, b in bounds:
            reduce_range(a, b)
            if consume:
                consume(a, b)
        return
    main = torch.cuda.current_stream(grads.g_z.device)
    produced = []
    for a, b in bounds:
        if produce:
            produce(a, b)
        ev = torch.cuda.Event()
        ev.record(main)
        produced.append(ev)
    reduced = []
    with torch.cuda.stream(comm_stream):
        for (a, b), ev in zip(bounds, produced):
            comm_stream.wait_event(ev)
            reduce_range(a, b)
            done = torch.cuda.Event()
            done.record(comm_stream)
            reduced.append(done)
    for (a, b), ev in zip(bounds, reduced):
        main.wait_event(ev)
        if consume:
            consume(a, b)


class ImageLoss:
    """Device image loss + pixel gradient (losses.py:103-113) for one image
    size; the value is read lazily (value() synchronises)."""

    def __init__(self, width: int, height: int, lambda_ssim: float, device):
        if lambda_ssim < 0:
            raise ValueError("lambda_ssim must be >= 0")
        if lambda_ssim > 0 and (width < 11 or height < 11):
            raise ValueError("images must be at least 11x11 for SSIM")  # losses.py:58-59
        self.W, self.H, self.lam = width, height, float(lambda_ssim)
        self.scratch = torch.empty(int(N.lib().ssg_loss_scratch_floats(width, height)), dtype=torch.float32,
                                   device=device)
        self.dL = torch.empty((height, width, 3), dtype=torch.float32, device=device)
        self.sums = torch.zeros(3, dtype=torch.float64, device=device)  # l1 sum, ssim sum, reg value

    def __call__(self, rendered: torch.Tensor, target: torch.Tensor) -> torch.Tensor:
        for t in (rendered, target):
            if tuple(t.shape) != (self.H, self.W, 3) or t.dtype != torch.float32 or not t.is_contiguous():
                raise ValueError("image dimensions differ")
        N.check(N.lib().ssg_image_loss(rendered.data_ptr(), target.data_ptr(), self.W, self.H, self.lam,
                                       self.scratch.data_ptr(), self.dL.data_ptr(), self.sums.data_ptr(),
                                       _stream(rendered.device)), "ssg_image_loss")
        return self.dL

    def value_tensor(self) -> torch.Tensor:
        """(1-l) L1 + l (1 - SSIM) + regularizer value, on the device."""
        l1 = self.sums[0] / (3.0 * self.W * self.H)
        if self.lam == 0.0:
            img = l1
        else:
            n = 3.0 * (self.W - 10) * (self.H - 10)
            img = (1.0 - self.lam) * l1 + self.lam * (1.0 - self.sums[1] / n)
        return img + self.sums[2]


class IntervalStats:
    """trainer.py:40-58 on the device (fp64 sums, fp32 max)."""

    def __init__(self, n: int, device):
        self.uv_sum = torch.zeros(n, dtype=torch.float64, device=device)
        self.z_max = torch.zeros(n, dtype=torch.float32, device=device)
        self.mu_sum = torch.zeros((n, 3), dtype=torch.float64, device=device)
        self.steps = 0

    def add(self, grads: DeviceGrads, views: int = 1, skip: torch.Tensor | None = None, rows: tuple | None = None):
        """`skip`: optional device int32 flag; nonzero = this step adds nothing
        (the caller then takes the `views` back, see Trainer).  `rows`
        = (a, b): only primitives [a, b) (the step's view count is then
        added by the caller, once)."""
        n = self.uv_sum.numel()
        if grads.g_uv.numel() != n:  # trainer.py:146 starts a new interval after densify
            raise ValueError(f"IntervalStats covers {n} primitives, gradients {grads.g_uv.numel()}")
        a, b = rows if rows is not None else (0, n)
        N.check(N.lib().ssg_interval_stats_add_ex(b - a, grads.g_uv[a:b].data_ptr(), grads.g_z[a:b].data_ptr(),
                                                  grads.d_mu[a:b].data_ptr(), self.uv_sum[a:b].data_ptr(),
                                                  self.z_max[a:b].data_ptr(), self.mu_sum[a:b].data_ptr(),
                                                  skip.data_ptr() if skip is not None else None,
                                                  _stream(self.uv_sum.device)), "ssg_interval_stats_add_ex")
        if rows is None:
            self.steps += views

    def bundle(self):
        tr = getattr(self, "_trainer", None)
        if tr is not None:  # a pipelined step may still owe its view-count correction
            tr.flush()
        d = max(self.steps, 1)
        return dataclasses.make_dataclass("Stats", ["g_uv", "g_z", "d_mu"])(
            self.uv_sum / d, self.z_max, self.mu_sum / d)


class DeviceAdam:
    """Adam state on the device (fp32 moments, one pair per scene field,
    adam.py:60-61) bound to a DeviceScene."""

    FIELDS = ("mu", "log_scale", "rot", "sh", "logits", "beta", "dir")

    def __init__(self, ds: DeviceScene, cfg: TrainConfig | None = None):
        self.ds = ds
        self.cfg = cfg or TrainConfig()
        self.t = 0
        self._alloc(ds.n)

    def _alloc(self, n: int):
        dev = self.ds.mu.device
        K = self.ds.K
        shapes = {"mu": (n, 3), "log_scale": (n, 3), "rot": (n, 4), "sh": (n, K, 3), "logits": (n, 2),
                  "beta": (n, 3), "dir": (n, 3)}
        self.m = {k: torch.zeros(s, dtype=torch.float32, device=dev) for k, s in shapes.items()}
        self.v = {k: torch.zeros_like(t) for k, t in self.m.items()}
        self.row_ok = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        self.n_skipped_dev = torch.zeros(1, dtype=torch.int32, device=dev)  # accumulated, adam.py:79

    def step(self, grads, iteration: int = 0, d_beta: torch.Tensor | None = None,
             skip: torch.Tensor | None = None, rows: tuple | None = None, advance: bool = True) -> None:
        """adam.py:71-97; `d_beta` (d_eta + regularizer) drives beta, d_eta
        drives dir.  `skip`: optional device int32 flag, nonzero = the step is
        skipped on the device (the caller then takes `t` back, see Trainer).
        `rows` = (a, b): update primitives [a, b) only (d_beta then covers
        the same rows); advance=False keeps the step count (the later ranges
        of one step: the caller advances once)."""
        ds, cfg = self.ds, self.cfg
        if ds.n == 0:
            return
        if advance:
            self.t += 1
        a, b = rows if rows is not None else (0, ds.n)
        if b <= a:
            return
        sub = ds.rows(a, b)
        p = N.SsgParams()
        p.n, p.sh_degree, p.sh_coeffs = b - a, ds.sh_degree, ds.K
        p.mu, p.log_scale, p.rot = sub.mu.data_ptr(), sub.log_scale.data_ptr(), sub.rot.data_ptr()
        p.sh, p.opacity_logits = sub.sh.data_ptr(), sub.opacity_logits.data_ptr()
        p.beta, p.dir = sub.beta.data_ptr(), sub.dir.data_ptr()
        g = N.SsgGradBuffers()  # any object with the gradient fields (row slices [a, b))
        g.d_mu, g.d_log_scale = grads.d_mu[a:b].data_ptr(), grads.d_log_scale[a:b].data_ptr()
        g.d_rot, g.d_sh = grads.d_rot[a:b].data_ptr(), grads.d_sh[a:b].data_ptr()
        g.d_opacity_logits, g.d_eta = grads.d_opacity_logits[a:b].data_ptr(), grads.d_eta[a:b].data_ptr()
        g.d_beta = d_beta.data_ptr() if d_beta is not None else None
        s = N.SsgAdamState()
        for f in self.FIELDS:
            setattr(s, "m_" + f, self.m[f][a:b].data_ptr())
            setattr(s, "v_" + f, self.v[f][a:b].data_ptr())
        s.row_ok, s.n_skipped = self.row_ok[a:b].data_ptr(), self.n_skipped_dev.data_ptr()
        hp = N.SsgAdamHparams()
        hp.t = self.t
        hp.lr_mu, hp.lr_scale, hp.lr_rot = cfg.position_lr_at(iteration), cfg.lr_scale, cfg.lr_rot
        hp.lr_sh, hp.lr_opacity, hp.lr_beta = cfg.lr_sh, cfg.lr_opacity, cfg.lr_beta
        hp.skip = skip.data_ptr() if skip is not None else None
        N.check(N.lib().ssg_adam_step(ctypes.byref(p), ctypes.byref(g), ctypes.byref(s), ctypes.byref(hp),
                                      _stream(ds.mu.device)), "ssg_adam_step")

    @property
    def n_skipped(self) -> int:
        """Primitive-steps skipped so far for a non-finite gradient (adam.py:79)."""
        return int(self.n_skipped_dev.item())


class Trainer:
    """Per-image-size scratch (loss, regularizer buffers) for training_step.

    pipelined=True runs each step without a host read-back: the finite-loss
    branch of fit2d.py:70-71 and the instance-capacity check become a device
    flag (0 run, 1 non-finite loss, 2 instance overflow; MAX over ranks) that
    Adam and the interval statistics consume, so the update is skipped on the
    device exactly when the synchronous step would skip it.  The flag is read
    back asynchronously and checked when the next step starts (or at
    flush()): a skipped step takes back the host's Adam step count and the
    statistics' view count, and an overflowed step (its lists were truncated,
    so its update was skipped) is re-run synchronously with grown buffers
    before anything else is queued -- the same parameters as the synchronous
    loop.  Call flush() before reading parameters (or the loss tensor of the
    last step) between steps."""

    def __init__(self, eng: Engine, ds: DeviceScene, adam: DeviceAdam, cfg: TrainConfig | None = None,
                 pipelined: bool = False, buckets: int = 1):
        self.eng, self.ds, self.adam = eng, ds, adam
        # buckets > 1: the projection backward, gradient all-reduce and the
        # update run per primitive range, the all-reduce of range i on a
        # communication stream under the projection backward of the later
        # ranges and the update of the earlier ones (bucketed_allreduce);
        # parameters are the same as with one bucket
        self.buckets = max(1, int(buckets))
        self._comm = None
        self.tail_events = None  # list: (start, end) CUDA events of each step's post-blend tail
        self.cfg = cfg or adam.cfg
        self._loss = {}
        self.d_beta = None
        self.pipelined = pipelined
        self._pending = None
        self._skip_dev = torch.zeros(1, dtype=torch.int32, device=eng.device)
        self._skip_host = torch.zeros(1, dtype=torch.int32, pin_memory=True) if pipelined else None
        self._loss_host = torch.zeros(1, dtype=torch.float64, pin_memory=True) if pipelined else None
        self.skipped_steps = 0  # pipelined steps skipped on the device (non-finite loss)
        if pipelined:
            adam._trainer = self  # densify_and_prune flushes through it

    def loss_for(self, W: int, H: int) -> ImageLoss:
        key = (W, H)
        if key not in self._loss:
            self._loss[key] = ImageLoss(W, H, self.cfg.lambda_ssim, self.eng.device)
        return self._loss[key]

    def loss_value(self) -> float:
        """The last pipelined step's loss on the host.  Waits only for that
        step's forward, loss and flag (read back right after the loss
        kernel), not for its backward and update, which keep running; a
        step flagged for a re-run (instance overflow) is resolved first and
        its re-run's loss returned."""
        if self._pending is None:
            raise RuntimeError("no pipelined step in flight")
        ev, _, loss = self._pending
        ev.synchronize()
        if int(self._skip_host[0]) == 2:
            self.flush()
            return float(loss)
        return float(self._loss_host[0])

    def flush(self) -> None:
        """Resolve the last pipelined step (see the class docstring)."""
        if self._pending is None:
            return
        ev, args, loss = self._pending
        self._pending = None
        ev.synchronize()
        code = int(self._skip_host[0])
        if code == 0:
            return
        view, target, iteration, stats, s, group = args
        self.adam.t -= 1  # the device skipped this step's update
        if stats is not None:
            stats.steps -= _world(group)
        if code == 1:  # non-finite loss: skipped, as fit2d.py:70-71
            self.skipped_steps += 1
            return
        try:  # instance overflow: grow the buffers and run the step for real
            self.eng.instances()
        except N.NativeError:
            pass
        redo, _ = self._step_sync(view, target, iteration, stats, s, group, True)
        loss.copy_(redo)  # the step's returned loss becomes the re-run's

    def _stage_target(self, target: torch.Tensor):
        """A host target image (pinned: asynchronous) goes up on a copy
        stream while the forward renders; _target_ready makes the loss wait
        for it.  Device targets pass through."""
        if target.is_cuda:
            return target, None
        st = getattr(self, "_h2d", None)
        if st is None:
            st = self._h2d = torch.cuda.Stream(self.eng.device)
        with torch.cuda.stream(st):
            t = target.to(self.eng.device, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
        return t, ev

    def _target_ready(self, staged) -> torch.Tensor:
        t, ev = staged
        if ev is not None:
            main = torch.cuda.current_stream(self.eng.device)
            main.wait_event(ev)
            t.record_stream(main)
        return t

    def step(self, view, target: torch.Tensor, iteration: int, stats: IntervalStats | None = None,
             s: float = 0.3, group=None, check_finite: bool = True):
        """fit2d.py:62-78.  Returns (loss tensor of this rank, frame).
        `target` may be a device tensor or a host one (pinned host memory
        uploads under the forward)."""
        if not self.pipelined:
            return self._step_sync(view, target, iteration, stats, s, group, check_finite)
        self.flush()
        eng, ds, cfg = self.eng, self.ds, self.cfg
        staged = self._stage_target(target)
        f = eng.forward(ds, view, s, sync=False)
        lossfn = self.loss_for(f.width, f.height)
        target = self._target_ready(staged)
        dL = lossfn(f.color, target)
        n = ds.n
        if self.d_beta is None or self.d_beta.shape[0] < n:
            self.d_beta = torch.empty((max(n, 1), 3), dtype=torch.float32, device=eng.device)
        self._penalty(lossfn)
        # the step's loss and fate on the device, one kernel: 2 overflow > 1
        # non-finite > 0 run
        v = torch.empty(1, dtype=torch.float64, device=eng.device)
        N.check(N.lib().ssg_step_value(lossfn.sums.data_ptr(), lossfn.W, lossfn.H, lossfn.lam,
                                       eng.n_inst_dev.data_ptr(), eng.capacity, v.data_ptr(),
                                       self._skip_dev.data_ptr(), _stream(eng.device)), "ssg_step_value")
        if _world(group) > 1:
            dist.all_reduce(self._skip_dev, op=dist.ReduceOp.MAX, group=group)
        # read the flag back now: waiting for it at the next step then waits
        # for this step's forward and loss only, not for its backward + Adam
        self._skip_host.copy_(self._skip_dev, non_blocking=True)
        self._loss_host.copy_(v, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        if stats is not None:
            stats._trainer = self  # bundle() flushes first
        self._update(view, s, f, dL, iteration, stats, group, self._skip_dev, lossfn)
        loss = v[0]  # this rank's loss (taken before the update, as fit2d.py:69 does)
        self._pending = (ev, (view, target, iteration, stats, s, group), loss)
        return loss, f

    def _penalty(self, lossfn):
        """sums[2] = the regularizer value (value-only ssg_regularize), so
        the finite-loss test sees loss + penalty as fit2d.py:69-71 does."""
        ds, cfg = self.ds, self.cfg
        N.check(N.lib().ssg_regularize(ds.n, ds.beta.data_ptr(), ds.opacity_logits.data_ptr(), None,
                                       cfg.lambda_beta_reg, cfg.lambda_opacity_reg, None, None,
                                       lossfn.sums.data_ptr(), _stream(self.eng.device)), "ssg_regularize")

    def _step_sync(self, view, target: torch.Tensor, iteration: int, stats: IntervalStats | None,
                   s: float, group, check_finite: bool):
        eng, ds, cfg = self.eng, self.ds, self.cfg
        staged = self._stage_target(target)
        f = eng.forward(ds, view, s, sync=False)  # M is checked with the loss below
        lossfn = self.loss_for(f.width, f.height)
        target = self._target_ready(staged)
        dL = lossfn(f.color, target)
        n = ds.n
        if self.d_beta is None or self.d_beta.shape[0] < n:
            self.d_beta = torch.empty((max(n, 1), 3), dtype=torch.float32, device=eng.device)
        # the regularizer value is part of the loss (losses.py:146-149); its
        # gradients are folded in after the backward and the statistics
        self._penalty(lossfn)
        v = lossfn.value_tensor()
        try:  # one read-back for the instance-count check and the loss value
            _, (loss,) = eng.instances(v)
        except N.NativeError:  # the scene outgrew the instance buffers: redo synchronised
            f = eng.forward(ds, view, s, sync=True)
            dL = lossfn(f.color, target)
            self._penalty(lossfn)
            v = lossfn.value_tensor()
            loss = float(v)
        if check_finite:
            # every rank must take the same branch (the all-reduce below is
            # collective): the step is skipped when any rank's view diverged
            bad = any_rank(not math.isfinite(loss), group, eng.device)
            if bad:  # fit2d.py:70-71: no backward, no update
                return v, f
        self._update(view, s, f, dL, iteration, stats, group, None, lossfn)
        return lossfn.value_tensor(), f

    def _comm_stream(self) -> torch.cuda.Stream:
        if self._comm is None:
            self._comm = torch.cuda.Stream(self.eng.device)
        return self._comm

    def _regularize(self, grads: DeviceGrads, rows: tuple, sums: torch.Tensor) -> None:
        """losses.py:116-136 gradients for primitives [a, b): d_beta = d_eta
        + the beta penalty's, d_logits += the opacity penalty's (after the
        all-reduce: the penalty is added once, not per rank)."""
        a, b = rows
        ds, cfg = self.ds, self.cfg
        N.check(N.lib().ssg_regularize(b - a, ds.beta[a:b].data_ptr(), ds.opacity_logits[a:b].data_ptr(),
                                       grads.d_eta[a:b].data_ptr(), cfg.lambda_beta_reg, cfg.lambda_opacity_reg,
                                       self.d_beta[a:b].data_ptr(), grads.d_opacity_logits[a:b].data_ptr(),
                                       sums.data_ptr(), _stream(self.eng.device)), "ssg_regularize")

    def _update(self, view, s, f, dL, iteration, stats, group, skip, lossfn) -> None:
        """Backward, gradient all-reduce, interval statistics, regularizer
        and Adam (fit2d.py:72-78, trainer.py:127-129 for the view-parallel
        sum), in one piece or per primitive bucket."""
        eng, ds = self.eng, self.ds
        n = ds.n
        world = _world(group)
        grads = eng.backward(ds, view, s, f.final_T, f.last_idx, dL, rebin=False, projection=False)
        cam = camera_struct(view, s)
        tail = None
        if self.tail_events is not None:  # the post-blend tail: projection backward .. Adam
            tail = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            tail[0].record()
            self.tail_events.append(tail)
        if self.buckets <= 1:
            eng.projection_backward(ds, cam, grads)
            allreduce_gradients(grads, group)
            if stats is not None:
                stats.add(grads, views=world, skip=skip)
            self._regularize(grads, (0, n), lossfn.sums)
            self.adam.step(grads, iteration, d_beta=self.d_beta[:n], skip=skip)
            if tail is not None:
                tail[1].record()
            return
        if stats is not None:
            stats.steps += world
        self.adam.t += 1
        if getattr(self, "_reg_sums", None) is None:  # the penalty value stays in lossfn.sums
            self._reg_sums = torch.zeros(3, dtype=torch.float64, device=eng.device)

        def produce(a, b):
            eng.projection_backward(ds, cam, grads, rows=(a, b))

        def consume(a, b):
            if stats is not None:
                stats.add(grads, skip=skip, rows=(a, b))
            self._regularize(grads, (a, b), self._reg_sums)
            self.adam.step(grads, iteration, d_beta=self.d_beta[a:b], skip=skip, rows=(a, b), advance=False)

        bucketed_allreduce(grads, bucket_bounds(n, self.buckets), group, produce, consume,
                           comm_stream=self._comm_stream() if world > 1 else None)
        if tail is not None:
            tail[1].record()


def training_step(eng: Engine, ds: DeviceScene, adam: DeviceAdam, view, target: torch.Tensor,
                  iteration: int = 0, stats: IntervalStats | None = None, s: float = 0.3,
                  group=None) -> torch.Tensor:
    """One view-parallel step (fit2d.py:62-78 + the gradient all-reduce).
    Returns the (device) loss of this rank."""
    tr = getattr(adam, "_step_trainer", None)
    if tr is None or tr.eng is not eng or tr.ds is not ds:
        tr = Trainer(eng, ds, adam)
        adam._step_trainer = tr
    loss, _ = tr.step(view, target, iteration, stats=stats, s=s, group=group)
    return loss
