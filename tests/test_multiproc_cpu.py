"""Multi-process host logic on CPU (gloo, world size 2): the gradient
all-reduce of the view-parallel training step (SUM of the packed buffer,
MAX of g_z) and the view sharding of config 4."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_18334_b200.engine import DeviceGrads
from paper_2605_18334_b200.train import allreduce_gradients, any_rank
from paper_2605_18334_b200.views import shard_views


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _grads(rank, n=37, K=4):
    g = torch.Generator().manual_seed(100 + rank)
    widths = (3, 3, 4, 3 * K, 2, 3, 1)
    flat = torch.randn(n * sum(widths), generator=g)
    views, off = [], 0
    for w in widths:
        views.append(flat[off:off + n * w])
        off += n * w
    return DeviceGrads(flat=flat, screen=torch.zeros(n, 12), d_mu=views[0].view(n, 3),
                       d_log_scale=views[1].view(n, 3), d_rot=views[2].view(n, 4), d_sh=views[3].view(n, K, 3),
                       d_opacity_logits=views[4].view(n, 2), d_eta=views[5].view(n, 3), g_uv=views[6].view(n),
                       g_z=torch.rand(n, generator=g))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = _grads(rank)
    allreduce_gradients(g)
    q.put((rank, g.flat.clone(), g.g_z.clone(), g.d_sh.clone()))
    dist.destroy_process_group()


def test_gradient_allreduce_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict()
    for _ in range(2):
        r, flat, gz, dsh = q.get(timeout=120)
        out[r] = (flat, gz, dsh)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = _grads(0), _grads(1)
    want_flat = a.flat + b.flat
    want_gz = torch.maximum(a.g_z, b.g_z)
    for r in range(2):
        torch.testing.assert_close(out[r][0], want_flat)
        torch.testing.assert_close(out[r][1], want_gz)
        torch.testing.assert_close(out[r][2], a.d_sh + b.d_sh)   # views alias the packed buffer
    assert torch.equal(out[0][0], out[1][0])                      # replicas stay identical


def test_allreduce_is_noop_single_process():
    g = _grads(0)
    before = g.flat.clone()
    allreduce_gradients(g)
    assert torch.equal(before, g.flat)


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 8), (10, 4), (3, 8)])
def test_shard_views_partitions(n, world):
    parts = [shard_views(n, r, world) for r in range(world)]
    flat = [i for p in parts for i in p]
    assert flat == list(range(n))
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1


def _worker_any(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # the training step's finite-loss decision is collective: one diverged
    # view makes every rank skip the step (no rank waits in the all-reduce)
    q.put((rank, any_rank(rank == 1), any_rank(False)))
    dist.destroy_process_group()


def test_any_rank_decision_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_any, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] is True and r[2] is False for r in res)
