"""bench.py --config 4 / --config 5 (BASELINE.json configs 4 and 5).

config 4: Mip-NeRF360-scale 3M skew Gaussians (G4 ball scene), 64 orbit
          views at 1297x840, forward only.  The 64-view batch is sharded by
          view over the ranks (contiguous blocks, no collective): strong
          scaling of a fixed batch; value = 64 / (max over ranks of the batch
          time) views/s.
config 5: view-parallel training step on a 2M G5 scene: per rank one view
          forward + L1 loss + backward, SUM all-reduce of the packed gradient
          buffer and MAX of g_z over NCCL, device Adam; value = views trained
          per second over all ranks (weak scaling: one view per rank per step).
Timing: CUDA events, max over ranks, nvidia-smi clocks sampled during the
timed region (see bench.py).
"""

from __future__ import annotations

import json
import os
import sys
import statistics
import time

import numpy as np

import bench as B

N4, W4, H4, V4 = 3_000_000, 1297, 840, 64
N5 = 2_000_000


def _setup(local, world):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        B.init_dist(torch, dist, local)
    return torch, dist


def _helpers(torch, dist, world):
    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return barrier, max_over_ranks


def _pinned_scene(torch, scene):
    from paper_2605_18334_b200.scene import Scene

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()
    return Scene(*(pinned(getattr(scene, f)) for f in Scene.ARRAY_FIELDS), background=scene.background,
                 sh_degree=scene.sh_degree)


def config4(args, rank, world, local):
    torch, dist = _setup(local, world)
    barrier, max_over_ranks = _helpers(torch, dist, world)
    from paper_2605_18334_b200.engine import DeviceScene, Engine
    from paper_2605_18334_b200.raster import render_forward
    from paper_2605_18334_b200.synthetic import ball_scene, orbit_views
    from paper_2605_18334_b200.views import render_views, shard_views

    scene = ball_scene(N4, seed=0)
    views = orbit_views(V4, radius=4.0, elevation=1.2, width=W4, height=H4, fov_x=0.9)
    mine = [views[i] for i in shard_views(V4, rank, world)]
    eng = Engine(torch.device("cuda", local))
    eng.keep_inst_tile = False  # introspection-only output
    # view lanes: engines on their own streams, so one view's latency-bound
    # binning overlaps another's blend (views.render_views)
    lanes = [eng] + [Engine(torch.device("cuda", local)) for _ in range(max(args.lanes, 1) - 1)]
    for e in lanes:
        e.keep_inst_tile = False
    ds = DeviceScene.from_host(scene)
    out = torch.empty((len(mine), H4, W4, 3), dtype=torch.float32, device="cuda")
    pairs = 0
    for v in mine:  # warm-up + per-view work count
        f = eng.forward(ds, v, 0.3)
        pairs += B.tile_pairs(f, eng.ranges, W4, H4)
    for _ in range(max(args.warmup, 3) - 1):
        render_views(ds, mine, engine=lanes, out=out)
    # the batch (every view's kernels on every lane, the streams' fork and
    # join) as one CUDA graph, captured after warm-up with no host round
    # trip inside; every kernel still runs every step, the launch gaps go
    launch = "graph"
    try:
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap):
            render_views(ds, mine, engine=lanes, out=out, check=False)
        torch.cuda.current_stream().wait_stream(cap)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph):
            render_views(ds, mine, engine=lanes, out=out, check=False)
        run_batch = graph.replay
    except RuntimeError as ex:
        print(f"CUDA graph capture failed ({ex}); timing eager launches", file=sys.stderr)
        launch = "eager"

        def run_batch():
            render_views(ds, mine, engine=lanes, out=out)
    used = lanes[:-(-len(mine) // 8)]  # engines that rendered a group of 8 views
    run_batch()
    for e in used:
        e.instances()  # the captured batch stayed inside the buffers
    barrier()
    clocks = B.ClockSampler(local)
    clocks.start()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start = time.perf_counter()
    e0.record()
    for _ in range(args.steps):
        run_batch()
    e1.record()
    barrier()
    for e in used:
        e.instances()
    clocks.mark(t_start, time.perf_counter())
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    # per-stage times from one separate, untimed batch on one lane (stage
    # events would perturb the timed loop; lanes overlap stages): totals over
    # the batch / views
    eng.stage_events = {}
    render_views(ds, mine, engine=eng, out=out)
    torch.cuda.synchronize()
    stage_ms = {k: sum(a.elapsed_time(b) for a, b in v) / max(len(mine), 1) for k, v in eng.stage_events.items()}
    eng.stage_events = None

    # e2e (1): the batch host API (views.render_views_host): the scene in
    # pinned host memory uploaded once per batch, the rank's views rendered
    # (same lanes), the f32 images back to host; median of 3 batches
    from paper_2605_18334_b200.views import render_views_host
    pscene = _pinned_scene(torch, scene)
    render_views_host(pscene, mine, lanes=len(lanes))
    bt = []
    for _ in range(3):
        barrier()
        t0 = time.perf_counter()
        render_views_host(pscene, mine, lanes=len(lanes))
        bt.append(time.perf_counter() - t0)
    e2e_batch_s = max_over_ranks(statistics.median(bt))
    # e2e (2): the reference-facing call per view (render_forward with the
    # scene in pinned host memory, uploaded per call; fp64 frame back to host)
    render_forward(pscene, mine[0])
    barrier()
    t0 = time.perf_counter()
    for v in mine:
        render_forward(pscene, v)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    scene_bytes = N4 * (3 + 3 + 4 + 48 + 2 + 3 + 3) * 8

    peaks = json.load(open(os.path.join(B.ROOT, "MEASURED_PEAKS.json")))
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    r_fp32 = n_sm * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    per_view_blend = stage_ms.get("blend_fwd", 0.0) * 1e-3
    ach = B.FP32_PER_PAIR["blend_fwd"] * pairs / max(len(mine), 1) / max(per_view_blend, 1e-9)
    result = {
        "metric": "config 4: 64-view forward batch, 3M skew Gaussians @1297x840, views/s",
        "value": V4 * 1000.0 / ms, "unit": "views/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (blend) / f64 (preprocess)", "data": "synthetic",
        "config": {"workload": "config 4: G4 ball scene, 3M skew Gaussians (SH3, fp32-rounded), "
                               "orbit_views(64, r=4, elev=1.2, 1297x840, fov 0.9), forward only",
                   "parallelism": f"views sharded x{world} (contiguous blocks, no collective); "
                                  f"{len(lanes)} view lanes per GPU (engines on their own streams)",
                   "launch": launch,
                   "l2": "inputs larger than L2 (scene 912 MB)"},
        "stage_ms_per_view": stage_ms,
        "roofline": {"bound": "fp32", "kernel": "k_blend_forward", "achieved": ach / 1e12,
                     "peak": r_fp32 / 1e12, "unit": "Tinstr/s (FP32 lane)", "frac": ach / r_fp32,
                     "traffic": None},
        "clocks": clk,
        "e2e": {"value": V4 / e2e_batch_s,
                "unit": "views/s", "h2d_bytes_per_step": scene_bytes,
                "d2h_bytes_per_step": len(mine) * H4 * W4 * 3 * 4,
                "path": "views.render_views_host: the fp64 host scene (pinned) uploaded once per 64-view batch, "
                        "the batch rendered on the device, the (V,H,W,3) f32 images back to host",
                "drop_in_per_view": {"value": V4 / e2e_s, "unit": "views/s",
                                     "h2d_bytes_per_step": len(mine) * scene_bytes,
                                     "d2h_bytes_per_step": len(mine) * H4 * W4 * (24 + 8 + 4 + 8),
                                     "path": "render_forward per view (the reference API: the scene uploaded per "
                                             "call), fp64 frame bundle back to host"}},
        # per view the frame's forward launches minus the projection (one
        # batched projection per 8 views)
        "gpu_launches": ((B.LAUNCHES_PER_FRAME - 4) * len(mine) + -(-len(mine) // 8)) * args.steps,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        sub_view = views[0]
        kind, run, desc = _cpu_forward_sample(scene, sub_view, 64)
        run()
        t0 = time.perf_counter()
        run()
        t = (time.perf_counter() - t0) * 64
        result["cpu_baseline"] = {"value": 1.0 / t, "unit": "views/s", "cores": B.cpu_cores(), "kind": kind,
                                  "sample": desc}
    if rank == 0:
        if B.SHARED_GPU:
            result["shared_gpu_test"] = True
        print(json.dumps(result))
    if world > 1:
        dist.destroy_process_group()


def _cpu_forward_sample(scene, view, k):
    from paper_2605_18334_b200.synthetic import homothetic_sample
    sub, sv = homothetic_sample(scene, view, k)
    ref = B._load_reference()
    desc = (f"homothetic 1/{k} sample of orbit view 0 (forward only): {len(sub)} primitives, "
            f"{sv.width}x{sv.height}; per-view time = {k} x sample time")
    if ref is not None:
        rf, _ = ref
        return "reference", (lambda: rf(sub, sv, 0.3, backend_name="cython")), desc
    from oracle import oracle as O
    O.set_num_threads(B.cpu_cores())
    return "port", (lambda: O.render_forward(sub, sv, 0.3)), desc


def _cpu_train_sample(scene, view, target, k):
    """The reference's fit2d.training_step (Cython rasterizer on all cores,
    SSIM loss, Adam) on a homothetic 1/k sample of one config-5 view."""
    from paper_2605_18334_b200.synthetic import homothetic_sample
    sub, sv = homothetic_sample(scene, view, k)
    ys = (np.arange(sv.height) * view.height) // sv.height
    xs = (np.arange(sv.width) * view.width) // sv.width
    tgt = target[ys][:, xs].astype(np.float64)
    desc = (f"homothetic 1/{k} sample of training view 0: {len(sub)} primitives, {sv.width}x{sv.height}, "
            f"target subsampled; per-step time = {k} x sample time")
    ref = B._load_reference()
    if ref is None:
        return None
    from skewsplat.fit2d import training_step as ref_step
    from skewsplat.optimize.adam import Adam
    from skewsplat.optimize.config import TrainConfig
    import skewsplat.scene as S
    rs = S.Scene(*(getattr(sub, f).copy() for f in sub.ARRAY_FIELDS), background=sub.background.copy(),
                 sh_degree=sub.sh_degree)
    cfg = TrainConfig()
    adam = Adam(rs, cfg)
    ref_step(rs, sv, tgt, cfg, adam, 0)
    t0 = time.perf_counter()
    ref_step(rs, sv, tgt, cfg, adam, 1)
    t = (time.perf_counter() - t0) * k
    return {"value": 1.0 / t, "unit": "views/s", "cores": B.cpu_cores(), "kind": "reference", "sample": desc}


def config5(args, rank, world, local):
    torch, dist = _setup(local, world)
    barrier, max_over_ranks = _helpers(torch, dist, world)
    from paper_2605_18334_b200.engine import DeviceScene, Engine
    from paper_2605_18334_b200.synthetic import ball_scene, fp32_round, orbit_views
    from paper_2605_18334_b200.train import DeviceAdam, Trainer

    target_scene = ball_scene(N5, seed=0)
    views = orbit_views(V4, radius=4.0, elevation=1.2, width=W4, height=H4, fov_x=0.9)
    eng = Engine(torch.device("cuda", local))
    eng.keep_inst_tile = False  # introspection-only output
    tgt_ds = DeviceScene.from_host(target_scene)
    targets = torch.empty((V4, H4, W4, 3), dtype=torch.float32, device="cuda")
    for i, v in enumerate(views):
        eng.forward(tgt_ds, v, 0.3, color_out=targets[i])
    del tgt_ds
    start = target_scene.copy()
    start.mu += np.random.default_rng(5).normal(size=start.mu.shape) * 0.01
    ds = DeviceScene.from_host(fp32_round(start))
    adam = DeviceAdam(ds)
    # pipelined steps: no host read-back inside a step (the finite-loss branch
    # and the instance check are a device flag, resolved at the next step)
    buckets = args.buckets if getattr(args, "buckets", None) else (4 if world > 1 else 1)
    tr = Trainer(eng, ds, adam, pipelined=True, buckets=buckets)
    step_no = [0]

    def step(target=None):
        i = (step_no[0] * world + rank) % V4
        step_no[0] += 1
        loss, _ = tr.step(views[i], targets[i] if target is None else target, i)
        return loss

    clocks = B.ClockSampler(local)
    clocks.start()
    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start = time.perf_counter()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    barrier()
    clocks.mark(t_start, time.perf_counter())
    clk = clocks.stop()
    tr.flush()
    assert tr.skipped_steps == 0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    # e2e: the step's input image from pinned host memory, loss read back
    host_t = torch.empty((H4, W4, 3), dtype=torch.float32, pin_memory=True)
    host_t.copy_(targets[0].cpu())
    # a run of steps timed whole (wall clock, everything finished at the end):
    # each step uploads its image and reads its loss back before the host
    # queues the next one
    n_e2e = max(args.e2e_steps, 10)
    step(host_t)
    tr.loss_value()
    barrier()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        step(host_t)  # uploaded by the trainer under the step's forward
        tr.loss_value()  # the loss back on the host; the backward and update keep running
    tr.flush()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / n_e2e)
    # the post-blend tail (projection backward, all-reduce, statistics,
    # regularizer, Adam) from separate untimed steps: what the bucketed
    # all-reduce can hide its communication under
    tr.tail_events = []
    for _ in range(3):
        step()
    tr.flush()
    torch.cuda.synchronize()
    tail_ms = statistics.median(a.elapsed_time(b) for a, b in tr.tail_events)
    tr.tail_events = None
    grad_bytes = int(eng.g_flat.numel() * 4 + eng.g_z.numel() * 4)
    busbw = 725e9  # 8-rank all-reduce bus bandwidth at 1 GiB, /opt/skills/guides/B200_PROFILING.md
    model = {}
    for nr in (2, 4, 8):
        comm = grad_bytes * 2 * (nr - 1) / nr / busbw * 1e3
        # ranges of equal size: range i's all-reduce overlaps the later ranges'
        # projection backward and the earlier ranges' update, so the step
        # grows by max(0, C - tail (B-1)/B) with B = 4
        exp4 = max(0.0, comm - tail_ms * 3 / 4)
        model[str(nr)] = {"comm_ms": comm, "exposed_ms_unbucketed": comm, "exposed_ms_4_buckets": exp4,
                          "step_frac_unbucketed": comm / (ms + comm), "step_frac_4_buckets": exp4 / (ms + exp4)}
    allreduce = {"bytes_per_rank": grad_bytes, "buckets": buckets, "tail_ms": tail_ms,
                 "model_busbw_gbs": busbw / 1e9, "model": model,
                 "note": "N = 1 measures the tail the communication can hide under; comm_ms = bytes x 2(N-1)/N / "
                         "bus bandwidth (not measured here: one GPU per lease)" if world == 1 else
                         "measured: ms_per_step includes the bucketed all-reduce"}
    result = {
        "metric": "config 5: view-parallel training step, 2M skew Gaussians @1297x840, views/s trained",
        "value": world * 1000.0 / ms, "unit": "views/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (blend, grads, moments) / f64 (preprocess)", "data": "synthetic",
        "config": {"workload": "config 5: G5 (ball scene, 2M), targets rendered from it, start perturbed "
                               "(mu + N(0, 0.01)); per step per rank (fit2d.training_step): fwd, "
                               "0.8 L1 + 0.2 (1 - SSIM) loss + pixel gradient, finite check, bwd, all-reduce, "
                               "interval stats, regularizers, Adam (TrainConfig defaults); pipelined: the "
                               "finite check and instance check are a device flag resolved at the next step",
                   "parallelism": f"view-parallel x{world}, NCCL all-reduce SUM of {N5 * 65 * 4 / 1e6:.0f} MB "
                                  "packed gradients + MAX of g_z"},
        "allreduce": allreduce,
        "clocks": clk,
        "e2e": {"value": world / e2e_s, "unit": "views/s", "h2d_bytes_per_step": H4 * W4 * 12,
                "d2h_bytes_per_step": 12, "path": "Trainer.step with the target image from pinned host "
                                                  "memory (uploaded under the forward) and the loss (fp64) "
                                                  "and step flag read back every step (Trainer.loss_value: "
                                                  "waits for the step's forward and loss, the backward and "
                                                  "update keep running under the next step's host work)"},
        # per step (tools/count_launches.py, torch.profiler): the frame's 22, image loss 2,
        # regularizer value + gradients 2, step value 1, Adam 9 (row check, 7 fields,
        # quaternion renorm) = 36
        "gpu_launches": (B.LAUNCHES_PER_FRAME + 14) * args.steps,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = _cpu_train_sample(start, views[0], targets[0].cpu().numpy(), 64)
    if rank == 0:
        if B.SHARED_GPU:
            result["shared_gpu_test"] = True
        print(json.dumps(result))
    if world > 1:
        dist.destroy_process_group()


def main(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = B.device_index()
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps({"impl": "reference", "unavailable":
                              f"--impl reference is defined for the headline config 2 only (got {args.config})"}))
        return
    (config4 if args.config == 4 else config5)(args, rank, world, local)
