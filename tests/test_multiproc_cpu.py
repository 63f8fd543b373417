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
    # numpy (pickled by value): torch tensors would be shared through a
    # socket of this process, which may exit before the parent reads them
    q.put((rank, g.flat.numpy().copy(), g.g_z.numpy().copy(), g.d_sh.numpy().copy()))
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
        out[r] = (torch.from_numpy(flat), torch.from_numpy(gz), torch.from_numpy(dsh))
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


def _worker_bucketed(rank, world, port, q, n, buckets):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_18334_b200.train import bucket_bounds, bucketed_allreduce
    src = _grads(rank, n=n)
    g = _grads(rank, n=n)
    g.flat.zero_()
    g.g_z.zero_()
    order = []

    def produce(a, b):  # a range's gradients appear only at its produce step
        order.append(("p", a, b))
        for f in DeviceGrads.SUM_FIELDS + ("g_z",):
            getattr(g, f)[a:b] = getattr(src, f)[a:b]

    seen = {}

    def consume(a, b):  # a consumer sees its rows fully reduced
        order.append(("c", a, b))
        seen[(a, b)] = (g.d_sh[a:b].numpy().copy(), g.g_z[a:b].numpy().copy())

    bounds = bucket_bounds(n, buckets, align=8)
    bucketed_allreduce(g, bounds, produce=produce, consume=consume)
    q.put((rank, bounds, order, g.flat.numpy().copy(), g.g_z.numpy().copy(), seen))  # numpy: by value
    dist.destroy_process_group()


@pytest.mark.parametrize("n,buckets", [(37, 3), (64, 1), (200, 4)])
def test_bucketed_allreduce_world2(n, buckets):
    """bucketed_allreduce (config 5's overlapped all-reduce, train.py):
    every range is produced before its reduction, consumed after it, in
    range order, and the result equals one all-reduce of everything."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_bucketed, args=(r, 2, port, q, n, buckets)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, bounds, order, flat, gz, seen = q.get(timeout=120)
        res[r] = (bounds, order, flat, gz, seen)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = _grads(0, n=n), _grads(1, n=n)
    for r in range(2):
        bounds, order, flat, gz, seen = res[r]
        assert bounds[0][0] == 0 and bounds[-1][1] == n and all(x[1] == y[0] for x, y in zip(bounds, bounds[1:]))
        assert len(bounds) == min(buckets, len(bounds)) and all(x[0] % 8 == 0 for x in bounds)
        prod = [o for o in order if o[0] == "p"]
        cons = [o for o in order if o[0] == "c"]
        assert [o[1:] for o in prod] == bounds and [o[1:] for o in cons] == bounds
        torch.testing.assert_close(torch.from_numpy(flat), a.flat + b.flat)
        torch.testing.assert_close(torch.from_numpy(gz), torch.maximum(a.g_z, b.g_z))
        for (lo, hi), (dsh, z) in seen.items():
            torch.testing.assert_close(torch.from_numpy(dsh), a.d_sh[lo:hi] + b.d_sh[lo:hi])
            torch.testing.assert_close(torch.from_numpy(z), torch.maximum(a.g_z[lo:hi], b.g_z[lo:hi]))
    assert (res[0][2] == res[1][2]).all()


@pytest.mark.parametrize("n,buckets", [(0, 4), (100, 1), (1000, 4), (1000, 16), (130, 8)])
def test_bucket_bounds(n, buckets):
    from paper_2605_18334_b200.train import bucket_bounds
    bounds = bucket_bounds(n, buckets)
    if n == 0:
        assert bounds == [(0, 0)]
        return
    assert bounds[0][0] == 0 and bounds[-1][1] == n
    assert all(lo < hi for lo, hi in bounds) and len(bounds) <= buckets
    assert all(lo % 128 == 0 for lo, _ in bounds)
