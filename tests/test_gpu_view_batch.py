"""View-batched projection (ssg_preprocess_forward_views / Engine.forward_views):
every per-view output equals the single-view kernel's bit for bit, for every SH
degree, batch sizes across the 8-view group boundary, primitives behind some
cameras, and block-ragged scene sizes; frames and a following backward equal the
one-view path.  The reference renders such batches one render_forward at a time
(trajectory.py:12-31)."""

import ctypes

import numpy as np
import pytest
import torch

from helpers import random_scene, random_view
from paper_2605_18334_b200 import _native as N
from paper_2605_18334_b200.engine import DeviceScene, Engine, camera_struct
from paper_2605_18334_b200.synthetic import ball_scene, fp32_round, orbit_views

pytestmark = pytest.mark.gpu

FIELDS = ("splat", "splat64", "depth_key", "tile_count", "tile_rect")


def _single_records(eng, ds, view):
    """What ssg_preprocess_forward writes for one view (fresh buffers)."""
    n = ds.n
    out = {f: torch.empty_like(getattr(eng, f)[:max(n, 1)]) for f in FIELDS}
    extra = dict(valid=torch.empty(max(n, 1), dtype=torch.uint8, device="cuda"),
                 depth=torch.empty(max(n, 1), dtype=torch.float64, device="cuda"),
                 radius=torch.empty(max(n, 1), dtype=torch.float64, device="cuda"),
                 nf=torch.zeros(1, dtype=torch.int32, device="cuda"))
    p = N.SsgPrimBuffers()
    p.splat, p.splat64, p.depth_key = (out[f].data_ptr() for f in ("splat", "splat64", "depth_key"))
    p.tile_count, p.tile_rect = out["tile_count"].data_ptr(), out["tile_rect"].data_ptr()
    p.valid, p.depth, p.radius = (extra[f].data_ptr() for f in ("valid", "depth", "radius"))
    p.n_skew_fallback = extra["nf"].data_ptr()
    cam = camera_struct(view, 0.3)
    sc = ds.struct()
    N.check(N.lib().ssg_preprocess_forward(ctypes.byref(sc), ctypes.byref(cam), ctypes.byref(p),
                                           torch.cuda.current_stream().cuda_stream), "ssg_preprocess_forward")
    return {f: t[:n] for f, t in out.items()}, int(extra["nf"].item())


def _batch_records(eng, ds, views):
    """ssg_preprocess_forward_views over `views`, all outputs (valid /
    depth / radius written too) in fresh buffers."""
    n, k = ds.n, len(views)
    sets, arr = [], (N.SsgPrimBuffers * k)()
    for j in range(k):
        d = {f: torch.empty_like(getattr(eng, f)[:max(n, 1)]) for f in FIELDS}
        d["valid"] = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
        d["depth"] = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
        d["radius"] = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
        d["nf"] = torch.full((1,), 7, dtype=torch.int32, device="cuda")  # the call zeroes it
        p = arr[j]
        p.splat, p.splat64, p.depth_key = (d[f].data_ptr() for f in ("splat", "splat64", "depth_key"))
        p.tile_count, p.tile_rect = d["tile_count"].data_ptr(), d["tile_rect"].data_ptr()
        p.valid, p.depth, p.radius = (d[f].data_ptr() for f in ("valid", "depth", "radius"))
        p.n_skew_fallback = d["nf"].data_ptr()
        sets.append(d)
    cams = (N.SsgCamera * k)(*[camera_struct(v, 0.3) for v in views])
    sc = ds.struct()
    N.check(N.lib().ssg_preprocess_forward_views(ctypes.byref(sc), cams, arr, k,
                                                 torch.cuda.current_stream().cuda_stream),
            "ssg_preprocess_forward_views")
    return sets


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
@pytest.mark.parametrize("k", [1, 3, 8])
def test_batch_records_equal_single_view(deg, k):
    rng = np.random.default_rng(10 + deg)
    n = 1000 + 37 * deg  # not a multiple of the 128-thread block
    ds = DeviceScene.from_host(fp32_round(random_scene(rng, n, sh_degree=deg)))
    # some cameras inside the cloud: primitives behind them are invalid
    views = [random_view(rng, 96 + 8 * j, 64, dist=(0.3 if j % 3 == 2 else 5.0)) for j in range(k)]
    eng = Engine()
    eng._ensure_prim(n)
    sets = _batch_records(eng, ds, views)
    for j, v in enumerate(views):
        ref, nf = _single_records(eng, ds, v)
        for f in FIELDS:
            assert torch.equal(sets[j][f][:n], ref[f]), (deg, k, j, f)
        eng.project(ds, v)
        assert torch.equal(sets[j]["valid"][:n], eng.valid[:n])
        assert torch.equal(sets[j]["depth"][:n], eng.depth[:n])
        assert torch.equal(sets[j]["radius"][:n], eng.radius[:n])
        assert int(sets[j]["nf"].item()) == nf


def test_batch_rejects_bad_arguments():
    rng = np.random.default_rng(3)
    ds = DeviceScene.from_host(fp32_round(random_scene(rng, 50)))
    eng = Engine()
    eng._ensure_prim(ds.n)
    views = [random_view(rng) for _ in range(N.MAX_BATCH_VIEWS + 1)]
    with pytest.raises(ValueError):
        _batch_records(eng, ds, views)  # more than SSG_MAX_BATCH_VIEWS
    big = random_view(rng, 70000, 64)
    with pytest.raises(ValueError, match="image dimension overflow"):
        _batch_records(eng, ds, [big])


def test_forward_views_frames_and_backward_equal_single():
    rng = np.random.default_rng(5)
    ds = DeviceScene.from_host(fp32_round(random_scene(rng, 4000, sh_degree=3)))
    views = [random_view(rng, 128, 96) for _ in range(11)]  # two groups: 8 + 3
    eng = Engine()
    singles = []
    for v in views:
        f = eng.forward(ds, v, 0.3)
        singles.append([t.clone() for t in (f.color, f.final_T, f.n_contrib, f.last_idx)])
    dL = torch.randn((96, 128, 3), device="cuda")
    g1 = eng.backward(ds, views[-1], 0.3, eng.final_T, eng.last_idx, dL, rebin=False, deterministic=True)
    g1 = g1.flat.clone()
    b = Engine()
    out = b.forward_views(ds, views, 0.3)
    b.instances()
    for j in range(len(views)):
        assert torch.equal(out[j], singles[j][0])
    # the engine's frame buffers and records are the last view's
    assert torch.equal(b.final_T, singles[-1][1])
    assert torch.equal(b.n_contrib, singles[-1][2])
    assert torch.equal(b.last_idx, singles[-1][3])
    g2 = b.backward(ds, views[-1], 0.3, b.final_T, b.last_idx, dL, rebin=False, deterministic=True)
    assert torch.equal(g1, g2.flat)
    # a single-view forward after a batch is unaffected
    f = b.forward(ds, views[2], 0.3)
    assert torch.equal(f.color, singles[2][0])


def test_forward_views_config4_sample_lists_bit_exact():
    """G4 sample (300k primitives, 8 orbit views): per-view instance lists
    of the batch path equal the one-view path's."""
    scene = ball_scene(300_000, seed=1)
    ds = DeviceScene.from_host(scene)
    views = orbit_views(8, radius=4.0, elevation=1.2, width=320, height=208, fov_x=0.9)
    eng, b = Engine(), Engine()
    b.keep_inst_tile = True
    out = b.forward_views(ds, views[:1], 0.3)  # warm the buffers
    for j, v in enumerate(views):
        f = eng.forward(ds, v, 0.3)
        ref = (f.color.clone(), eng.inst_prim[:eng.last_m].clone(), eng.ranges.clone())
        out = b.forward_views(ds, [views[i] for i in range(j + 1)], 0.3)
        m = b.instances()
        assert m == eng.last_m
        assert torch.equal(out[j], ref[0])
        assert torch.equal(b.inst_prim[:m], ref[1])
        assert torch.equal(b.ranges, ref[2])


def test_render_views_host_equals_device_batch():
    from paper_2605_18334_b200.serving import quantize_u8_device
    from paper_2605_18334_b200.views import render_views, render_views_host
    rng = np.random.default_rng(9)
    scene = fp32_round(random_scene(rng, 3000, sh_degree=3))
    views = [random_view(rng, 112, 80) for _ in range(19)]
    ds = DeviceScene.from_host(scene)
    ref = render_views(ds, views, engine=Engine())
    for lanes in (1, 3):
        got = render_views_host(scene, views, lanes=lanes)
        assert got.dtype == np.float32 and got.shape == (19, 80, 112, 3)
        assert np.array_equal(got, ref.cpu().numpy())
    u8 = render_views_host(scene, views, lanes=2, u8=True)
    assert u8.dtype == np.uint8 and np.array_equal(u8, quantize_u8_device(ref).cpu().numpy())


def test_forward_views_empty_and_behind_camera_scenes():
    """No primitives, or every primitive behind the cameras: the batch
    renders the background, like the one-view path."""
    from paper_2605_18334_b200.scene import Scene
    rng = np.random.default_rng(4)
    views = [random_view(rng, 64, 48) for _ in range(10)]
    empty = Scene(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 4, 3)), np.zeros((0, 2)),
                  np.zeros((0, 3)), np.zeros((0, 3)), background=np.array([0.25, 0.5, 0.75]), sh_degree=1)
    eng = Engine()
    out = eng.forward_views(DeviceScene.from_host(empty), views, 0.3)
    eng.instances()
    assert torch.all(out == torch.tensor([0.25, 0.5, 0.75], device="cuda"))
    scene = fp32_round(random_scene(rng, 500, sh_degree=1))
    ds = DeviceScene.from_host(scene)
    behind = [random_view(rng, 64, 48, dist=0.01) for _ in range(3)]   # inside the cloud
    single = Engine()
    ref = [single.forward(ds, v, 0.3).color.clone() for v in behind]
    got = Engine().forward_views(ds, behind, 0.3)
    for a, b in zip(ref, got):
        assert torch.equal(a, b)


def test_render_views_host_speculation_is_exact():
    """A host batch of the scene the engine rendered last renders on the
    kept device copy while the upload runs, then checks the upload bitwise;
    a changed scene (one value of the last primitive) re-renders."""
    from paper_2605_18334_b200.views import lane_engines, render_views, render_views_host
    rng = np.random.default_rng(12)
    scene = fp32_round(random_scene(rng, 2500, sh_degree=2))
    views = [random_view(rng, 96, 72) for _ in range(11)]
    ref = render_views(DeviceScene.from_host(scene), views, engine=Engine()).cpu().numpy()
    render_views_host(scene, views, lanes=2)
    kept = lane_engines(2)[0]._host_batch_scene
    got = render_views_host(scene, views, lanes=2)
    assert lane_engines(2)[0]._host_batch_scene is kept          # speculation held
    assert np.array_equal(got, ref)
    moved = scene.copy()
    moved.sh[-1, 0, 0] += 0.25
    ref2 = render_views(DeviceScene.from_host(moved), views, engine=Engine()).cpu().numpy()
    got2 = render_views_host(moved, views, lanes=2)
    assert lane_engines(2)[0]._host_batch_scene is not kept      # caught, re-rendered
    assert np.array_equal(got2, ref2)
    moved.mu[-1, 0] += 1e-9                                       # fp64 geometry, one ulp-scale change
    ref3 = render_views(DeviceScene.from_host(moved), views, engine=Engine()).cpu().numpy()
    k2 = lane_engines(2)[0]._host_batch_scene
    assert np.array_equal(render_views_host(moved, views, lanes=2, u8=False), ref3)
    assert lane_engines(2)[0]._host_batch_scene is not k2
