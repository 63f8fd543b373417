"""Multi-view training loop on the device (reference trainer.py:89-153).

fit_multiview keeps the reference's contract -- one training view per
iteration drawn by the seeded RNG (rng.integers over the training split),
the densification cadence (densify_start <= it <= densify_end, every
densify_interval iterations, max_radii from the projection of the current
view when max_screen_radius is set), the interval statistics recreated after
every controller run, the log entries (iteration, loss, psnr, n_primitives
and the clone / split / prune counts since the last entry), the early stop
with a RuntimeWarning on a non-finite loss, and held-out PSNR / SSIM -- with
every step on the GPU: Trainer.step (render, L1 + SSIM loss and its pixel
gradient, backward, regularizers, Adam), densify_and_prune on the device
scene, metrics from the device loss kernel (the SSIM of losses.py:44-101 is
the metric's, metrics.py:42-45).  The backward runs in the deterministic
mode, so a seeded re-run is bitwise identical (reference test_trainer.py:
74-82).

init_multiview_scene restates trainer.py:60-77 + initialize.py:22-56 on the
host (same RNG draws, so the seeded runs start from the reference's scene).
"""

from __future__ import annotations

import dataclasses
import json
import math
import warnings

import numpy as np
import torch

from .engine import DeviceScene, Engine
from .scene import Scene
from .train import DeviceAdam, ImageLoss, IntervalStats, TrainConfig, Trainer

SH_C0 = 0.28209479177387814
INIT_OPACITY = 0.1            # initialize.py:19
TEST_EVERY = 8                # dataset.py:24
PSNR_CAP = 100.0              # metrics.py


@dataclasses.dataclass
class Dataset:
    """dataset.py:116-136: (image, view) pairs, every TEST_EVERY-th held out."""
    images: list

    def __post_init__(self):
        if len(self.train) < 1:
            raise ValueError("dataset must keep at least one training image")

    @property
    def test_indices(self) -> list[int]:
        return list(range(0, len(self.images), TEST_EVERY))

    @property
    def train(self) -> list:
        skip = set(self.test_indices)
        return [pair for i, pair in enumerate(self.images) if i not in skip]

    @property
    def test(self) -> list:
        return [self.images[i] for i in self.test_indices]


@dataclasses.dataclass
class TrainResult:
    scene: Scene
    log: list
    test_psnr: float | None
    test_ssim: float | None
    diverged_at: int | None
    n_skipped: int


def nn_log_scales(mu: np.ndarray, fallback: float = 0.1) -> np.ndarray:
    """initialize.py:22-31: isotropic log scales from nearest-neighbour distances."""
    n = mu.shape[0]
    if n < 2:
        d = np.full(max(n, 0), fallback)
    else:
        from scipy.spatial import cKDTree
        dist, _ = cKDTree(mu).query(mu, k=2)
        d = np.clip(dist[:, 1], 1e-4, None)
    return np.repeat(np.log(d)[:, None], 3, axis=1)


def initial_scene(mu, colors, background, sh_degree: int = 0) -> Scene:
    """initialize.py:34-56."""
    mu = np.asarray(mu, dtype=np.float64).reshape(-1, 3)
    colors = np.asarray(colors, dtype=np.float64).reshape(-1, 3)
    n = mu.shape[0]
    k = (sh_degree + 1) ** 2
    sh = np.zeros((n, k, 3))
    sh[:, 0, :] = (colors - 0.5) / SH_C0
    logit = math.log(INIT_OPACITY / (1.0 - INIT_OPACITY))
    return Scene(mu=mu, log_scale=nn_log_scales(mu), rot=np.tile([1.0, 0.0, 0.0, 0.0], (n, 1)), sh=sh,
                 opacity_logits=np.full((n, 2), logit), beta=np.zeros((n, 3)), dir=np.zeros((n, 3)),
                 background=background, sh_degree=sh_degree)


def init_multiview_scene(dataset, n_init: int, sh_degree: int, rng: np.random.Generator) -> Scene:
    """trainer.py:60-77: positions uniform in the unit box, background the
    per-channel median of the training pixels, colours their mean."""
    pixels = np.concatenate([np.asarray(img).reshape(-1, 3) for img, _ in dataset.train], axis=0)
    background = np.median(pixels, axis=0)
    mean_color = pixels.mean(axis=0)
    positions = rng.uniform(-1.0, 1.0, (n_init, 3))
    colors = np.tile(mean_color, (n_init, 1))
    return initial_scene(positions, colors, background=background, sh_degree=sh_degree)


def _host_scene(ds: DeviceScene) -> Scene:
    f64 = lambda t: t.detach().to(torch.float64).cpu().numpy()  # noqa: E731
    return Scene(mu=f64(ds.mu), log_scale=f64(ds.log_scale), rot=f64(ds.rot), sh=f64(ds.sh),
                 opacity_logits=f64(ds.opacity_logits), beta=f64(ds.beta), dir=f64(ds.dir),
                 background=np.array(ds.background), sh_degree=ds.sh_degree)


class _Images:
    """Device copies of the dataset images (uploaded once)."""

    def __init__(self, device):
        self.device, self.cache = device, {}

    def __call__(self, img) -> torch.Tensor:
        key = id(img)
        if key not in self.cache:
            self.cache[key] = (img, torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).to(self.device))
        return self.cache[key][1]


def _psnr(color: torch.Tensor, target: torch.Tensor) -> float:
    """metrics.py:33-39."""
    mse = float(((color.double() - target.double()) ** 2).mean())
    if mse == 0.0:
        return PSNR_CAP
    return float(min(10.0 * math.log10(1.0 / mse), PSNR_CAP))


def evaluate(eng: Engine, ds: DeviceScene, pairs, images: _Images) -> tuple[float, float]:
    """trainer.py:80-84: mean PSNR / SSIM of the renders against (image, view)."""
    ps, ss = [], []
    for img, view in pairs:
        f = eng.forward(ds, view, 0.3)
        tgt = images(img)
        ps.append(_psnr(f.color, tgt))
        lf = ImageLoss(f.width, f.height, 1.0, eng.device)
        lf(f.color, tgt)
        ss.append(float(lf.sums[1]) / (3.0 * (f.width - 10) * (f.height - 10)))
    return float(np.mean(ps)), float(np.mean(ss))


def fit_multiview(dataset, cfg: TrainConfig | None = None, n_init: int = 100, sh_degree: int = 0,
                  skew_enabled: bool = True, densify: bool = True, log_every: int = 100, log_stream=None,
                  device=None, step_fn=None) -> TrainResult:
    """trainer.py:89-153 on the GPU.  `step_fn` (tests): replaces the
    training step, called as step_fn(trainer, view, target, iteration,
    stats) -> (loss value, frame) like trainer_mod.training_step."""
    from .densify import densify_and_prune
    cfg = dataclasses.replace(cfg) if cfg is not None else TrainConfig()
    if not skew_enabled:
        cfg.lr_beta = 0.0
    cfg.validate()
    if n_init < 1:
        raise ValueError("n_init must be >= 1")
    rng = np.random.default_rng(cfg.seed)
    train = dataset.train
    scene = init_multiview_scene(dataset, n_init, sh_degree, rng)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    eng = Engine(dev)
    eng.deterministic = True       # bit-reproducible seeded runs, like the reference
    ds = DeviceScene.from_host(scene, dev)
    adam = DeviceAdam(ds, cfg)
    trainer = Trainer(eng, ds, adam, cfg)
    stats = IntervalStats(ds.n, dev)
    images = _Images(dev)

    def step(view, target, it, st):
        loss, frame = trainer.step(view, target, it, stats=st)
        return float(loss), frame

    step_fn = step_fn or (lambda tr, view, target, it, st: step(view, target, it, st))
    log: list = []
    counts = {"n_cloned": 0, "n_split": 0, "n_pruned": 0}
    diverged_at = None

    def emit(iteration, value, frame_psnr):
        entry = {"iteration": iteration, "loss": float(value), "psnr": frame_psnr, "n_primitives": ds.n,
                 **counts}
        log.append(entry)
        if log_stream is not None:
            log_stream.write(json.dumps(entry) + "\n")
            log_stream.flush()
        for key in counts:
            counts[key] = 0

    for it in range(cfg.iterations):
        img, view = train[rng.integers(len(train))]
        target = images(img)
        value, frame = step_fn(trainer, view, target, it, stats)
        if it % log_every == 0:
            emit(it, value, _psnr(frame.color, target))
        if not math.isfinite(value):
            warnings.warn(f"loss went non-finite at iteration {it}; stopping early", RuntimeWarning, stacklevel=2)
            diverged_at = it
            break
        if (densify and it > 0 and cfg.densify_start <= it <= cfg.densify_end
                and it % cfg.densify_interval == 0 and stats.steps > 0):
            max_radii = None
            if cfg.max_screen_radius is not None:
                max_radii = eng.project(ds, view, 0.3).clone()
            report = densify_and_prune(ds, stats.bundle(), cfg, adam=adam, max_radii=max_radii)
            for key in counts:
                counts[key] += report[key]
            stats = IntervalStats(ds.n, dev)

    test_psnr = test_ssim = None
    if dataset.test:
        test_psnr, test_ssim = evaluate(eng, ds, dataset.test, images)
    return TrainResult(scene=_host_scene(ds), log=log, test_psnr=test_psnr, test_ssim=test_ssim,
                       diverged_at=diverged_at, n_skipped=adam.n_skipped)
