"""Frame serving against the reference (oracle/_ref):
quantize_u8 byte-exact on identical fp64 input; render_frame payloads and
trajectory PNGs equal up to fp32-blend rounding (header exact, >= 99.9 % of
pixel bytes identical, the rest off by one)."""

import os
import sys

import numpy as np
import pytest

from helpers import random_scene, random_view
from paper_2605_18334_b200.serving import (HEADER, load_trajectory, quantize_u8, render_frame, render_trajectory,
                                           render_views_u8, save_trajectory)
from paper_2605_18334_b200.synthetic import fp32_round

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref():
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "skewsplat")):
        pytest.skip("oracle/_ref not present")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import skewsplat.dataset as D
    import skewsplat.service as SV
    import skewsplat.trajectory as TR
    return D, SV, TR


def test_quantize_u8_is_byte_exact():
    D, _, _ = _ref()
    rng = np.random.default_rng(0)
    img = rng.uniform(-0.2, 1.2, (97, 131, 3))
    img[0, :8, 0] = [k / 255.0 + 0.5 / 255.0 for k in range(8)]  # halfway cases
    img[1, :4, 1] = [0.5, 0.0, 1.0, 127.5 / 255.0]
    np.testing.assert_array_equal(quantize_u8(img), D.quantize_u8(img))
    with pytest.raises(ValueError):
        quantize_u8(np.zeros((4, 4)))


def _close_bytes(a: bytes, b: bytes):
    x, y = np.frombuffer(a, np.uint8).astype(int), np.frombuffer(b, np.uint8).astype(int)
    assert x.shape == y.shape
    d = np.abs(x - y)
    assert d.max() <= 1 and np.mean(d == 0) >= 0.999, (d.max(), np.mean(d == 0))


def test_render_frame_payload_matches_reference():
    _, SV, _ = _ref()
    rng = np.random.default_rng(5)
    scene = fp32_round(random_scene(rng, 400, sh_degree=1))
    view = random_view(rng, 96, 64)
    got, want = render_frame(scene, 42, view), SV.render_frame(scene, 42, view)
    assert got[:HEADER.size] == want[:HEADER.size]
    _close_bytes(got[HEADER.size:], want[HEADER.size:])


def test_trajectory_pngs_match_reference(tmp_path):
    D, _, TR = _ref()
    rng = np.random.default_rng(6)
    scene = fp32_round(random_scene(rng, 300, sh_degree=2))
    views = [random_view(rng, 64, 48) for _ in range(3)]
    save_trajectory(tmp_path / "traj.json", views)
    back = load_trajectory(tmp_path / "traj.json")
    assert len(back) == 3 and all(np.array_equal(a.c2w, b.c2w) for a, b in zip(back, views))
    ours = render_trajectory(scene, str(tmp_path / "traj.json"), tmp_path / "ours")
    import skewsplat.scene as S
    ref_scene = S.Scene(*(getattr(scene, f).copy() for f in scene.ARRAY_FIELDS), background=scene.background.copy(),
                        sh_degree=scene.sh_degree)
    theirs = TR.render_trajectory(ref_scene, views, tmp_path / "theirs")
    assert [os.path.basename(p) for p in ours] == [os.path.basename(p) for p in theirs]
    for a, b in zip(ours, theirs):
        _close_bytes(D.quantize_u8(D.load_image(a)).tobytes(), D.quantize_u8(D.load_image(b)).tobytes())
    batch = render_views_u8(scene, views)
    assert tuple(batch.shape) == (3, 48, 64, 3)
    _close_bytes(batch[0].cpu().numpy().tobytes(), D.quantize_u8(D.load_image(theirs[0])).tobytes())


def test_trajectory_batches_mixed_sizes_equal_per_view(tmp_path):
    """render_trajectory renders runs of one image size as device batches
    and encodes on a thread pool: files, names and pixels equal a per-view
    render, across a change of image size."""
    from PIL import Image

    from paper_2605_18334_b200.engine import DeviceScene, Engine
    from paper_2605_18334_b200.serving import quantize_u8_device
    rng = np.random.default_rng(9)
    scene = fp32_round(random_scene(rng, 500, sh_degree=1))
    views = [random_view(rng, 64, 48) for _ in range(5)] + [random_view(rng, 80, 40) for _ in range(4)] + \
        [random_view(rng, 64, 48)]
    paths = render_trajectory(scene, views, tmp_path / "t")
    assert [os.path.basename(p) for p in paths] == [f"{i:04d}.png" for i in range(len(views))]
    eng, ds = Engine(), DeviceScene.from_host(scene)
    for p, v in zip(paths, views):
        ref = quantize_u8_device(eng.forward(ds, v, 0.3).color).cpu().numpy()
        assert np.array_equal(np.asarray(Image.open(p).convert("RGB")), ref)
