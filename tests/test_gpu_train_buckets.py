"""Bucketed training update (Trainer(buckets=B)): the projection backward,
gradient all-reduce, interval statistics, regularizer and Adam run per
primitive range so that range i's all-reduce overlaps the later ranges'
projection backward and the earlier ranges' update (train.bucketed_allreduce,
config 5).  Row-local work, so the parameters must equal the one-bucket
step's bit for bit (deterministic gradients); the 2-GPU NCCL case (skipped on
a 1-GPU host) checks the view-parallel sum against a single process."""

import os
import socket

import numpy as np
import pytest
import torch

from helpers import random_scene, random_view
from paper_2605_18334_b200.engine import DeviceScene, Engine
from paper_2605_18334_b200.synthetic import fp32_round
from paper_2605_18334_b200.train import DeviceAdam, IntervalStats, TrainConfig, Trainer

pytestmark = pytest.mark.gpu
FIELDS = ("mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir")


def _setup(seed=3, n=1500):
    rng = np.random.default_rng(seed)
    target_scene = fp32_round(random_scene(rng, n, sh_degree=3))
    views = [random_view(rng, 96, 80) for _ in range(3)]
    eng = Engine()
    tds = DeviceScene.from_host(target_scene)
    targets = [eng.forward(tds, v, 0.3).color.clone() for v in views]
    start = target_scene.copy()
    start.mu += rng.normal(size=start.mu.shape) * 0.02
    return fp32_round(start), views, targets


def _run(start, views, targets, buckets, pipelined, steps=6):
    eng = Engine()
    eng.deterministic = True
    ds = DeviceScene.from_host(start)
    cfg = TrainConfig()
    cfg.lambda_beta_reg, cfg.lambda_opacity_reg = 1e-3, 1e-3  # the regularizer runs per range too
    adam = DeviceAdam(ds, cfg)
    stats = IntervalStats(ds.n, eng.device)
    tr = Trainer(eng, ds, adam, pipelined=pipelined, buckets=buckets)
    losses = []
    for it in range(steps):
        v, _ = tr.step(views[it % 3], targets[it % 3], it, stats=stats)
        losses.append(v)
    tr.flush()
    torch.cuda.synchronize()
    return ds, adam, stats, [float(x) for x in losses]


@pytest.mark.parametrize("pipelined", [False, True])
@pytest.mark.parametrize("buckets", [4, 7])
def test_buckets_equal_one_bucket_bitwise(buckets, pipelined):
    start, views, targets = _setup()
    a = _run(start, views, targets, 1, pipelined)
    b = _run(start, views, targets, buckets, pipelined)
    for f in FIELDS:
        assert torch.equal(getattr(a[0], f), getattr(b[0], f)), f
        if f != "opacity_logits":
            key = {"log_scale": "log_scale", "sh": "sh", "mu": "mu", "rot": "rot", "beta": "beta", "dir": "dir"}[f]
            assert torch.equal(a[1].m[key], b[1].m[key]) and torch.equal(a[1].v[key], b[1].v[key]), f
    assert a[1].t == b[1].t
    assert torch.equal(a[2].uv_sum, b[2].uv_sum) and torch.equal(a[2].z_max, b[2].z_max)
    assert torch.equal(a[2].mu_sum, b[2].mu_sum) and a[2].steps == b[2].steps
    # the loss carries the penalty value, an fp64 atomic sum (order-dependent in the last ulp)
    np.testing.assert_allclose(a[3], b[3], rtol=1e-12)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _no_reg():
    cfg = TrainConfig()
    cfg.lambda_beta_reg = cfg.lambda_opacity_reg = 0.0  # the reference below sums raw gradients
    return cfg


def _nccl_worker(rank, world, port, start, views, targets, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    eng = Engine(torch.device("cuda", rank))
    eng.deterministic = True
    ds = DeviceScene.from_host(start, eng.device)
    adam = DeviceAdam(ds, _no_reg())
    tr = Trainer(eng, ds, adam, buckets=4)
    for it in range(3):  # rank r trains view r of step it, the targets of rank r
        tr.step(views[(it + rank) % 3], targets[(it + rank) % 3].to(eng.device), it)
    torch.cuda.synchronize()
    q.put((rank, {f: getattr(ds, f).cpu() for f in FIELDS}))
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_nccl_two_ranks_match_summed_gradients():
    import torch.multiprocessing as mp
    start, views, targets = _setup(n=800)
    targets = [t.cpu() for t in targets]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, start, views, targets, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for f in FIELDS:  # replicas stay identical
        assert torch.equal(res[0][f], res[1][f]), f
    # one process: the two views' gradients summed, then the same updates
    eng = Engine()
    eng.deterministic = True
    ds = DeviceScene.from_host(start)
    adam = DeviceAdam(ds, _no_reg())
    from paper_2605_18334_b200.train import ImageLoss
    for it in range(3):
        acc = None
        for r in range(2):
            v = views[(it + r) % 3]
            f = eng.forward(ds, v, 0.3)
            lossfn = ImageLoss(f.width, f.height, adam.cfg.lambda_ssim, eng.device)
            dL = lossfn(f.color, targets[(it + r) % 3].cuda())
            g = eng.backward(ds, v, 0.3, f.final_T, f.last_idx, dL, rebin=False)
            acc = (g.flat.clone(), g.g_z.clone()) if acc is None else (acc[0] + g.flat, torch.maximum(acc[1], g.g_z))
        g.flat.copy_(acc[0])
        g.g_z.copy_(acc[1])
        adam.step(g, it)
    for f in FIELDS:
        torch.testing.assert_close(res[0][f], getattr(ds, f).cpu(), rtol=1e-5, atol=1e-6)


def _gloo_cuda_worker(rank, world, port, start, views, targets, q):
    """Two ranks on one GPU with gloo over CUDA tensors: exercises the
    comm-stream path of bucketed_allreduce (events, the grouped all-reduce,
    the per-range consumers) where NCCL needs one GPU per rank."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = Engine(torch.device("cuda", 0))
    eng.deterministic = True
    ds = DeviceScene.from_host(start, eng.device)
    adam = DeviceAdam(ds, _no_reg())
    tr = Trainer(eng, ds, adam, buckets=4)
    for it in range(3):
        tr.step(views[(it + rank) % 3], targets[(it + rank) % 3].to(eng.device), it)
    torch.cuda.synchronize()
    q.put((rank, {f: getattr(ds, f).cpu().numpy() for f in FIELDS}))
    dist.destroy_process_group()


def test_bucketed_allreduce_two_ranks_one_gpu_gloo():
    import torch.multiprocessing as mp
    start, views, targets = _setup(n=800)
    targets = [t.cpu() for t in targets]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_cuda_worker, args=(r, 2, port, start, views, targets, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for f in FIELDS:
        assert np.array_equal(res[0][f], res[1][f]), f
    # one process: the two views' gradients summed, then the same updates
    eng = Engine()
    eng.deterministic = True
    ds = DeviceScene.from_host(start)
    adam = DeviceAdam(ds, _no_reg())
    from paper_2605_18334_b200.train import ImageLoss
    for it in range(3):
        acc = None
        for r in range(2):
            v = views[(it + r) % 3]
            f = eng.forward(ds, v, 0.3)
            lossfn = ImageLoss(f.width, f.height, adam.cfg.lambda_ssim, eng.device)
            dL = lossfn(f.color, targets[(it + r) % 3].cuda())
            g = eng.backward(ds, v, 0.3, f.final_T, f.last_idx, dL, rebin=False)
            acc = (g.flat.clone(), g.g_z.clone()) if acc is None else (acc[0] + g.flat, torch.maximum(acc[1], g.g_z))
        g.flat.copy_(acc[0])
        g.g_z.copy_(acc[1])
        adam.step(g, it)
    for f in FIELDS:
        np.testing.assert_allclose(res[0][f], getattr(ds, f).cpu().numpy(), rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("pipelined", [False, True])
def test_host_targets_equal_device_targets(pipelined):
    """A pinned host target image uploads on the trainer's copy stream under
    the forward; the steps equal those with the image already on the device."""
    start, views, targets = _setup(seed=5, n=900)
    host = [t.cpu().pin_memory() for t in targets]
    a = _run(start, views, targets, 1, pipelined)
    b = _run(start, views, host, 1, pipelined)
    for f in FIELDS:
        assert torch.equal(getattr(a[0], f), getattr(b[0], f)), f
    np.testing.assert_allclose(a[3], b[3], rtol=1e-12)  # fp64 atomic loss sums: order-dependent ulps


def test_loss_value_equals_the_step_loss():
    """Trainer.loss_value (the pinned read-back right after the loss kernel)
    equals the step's returned device loss."""
    start, views, targets = _setup(seed=8, n=700)
    eng = Engine()
    ds = DeviceScene.from_host(start)
    tr = Trainer(eng, ds, DeviceAdam(ds), pipelined=True)
    for it in range(4):
        loss, _ = tr.step(views[it % 3], targets[it % 3], it)
        got = tr.loss_value()
        assert got == float(loss.item())
    tr.flush()
