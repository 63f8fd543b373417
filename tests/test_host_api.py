"""Host-side contract of the drop-in API (no GPU needed): argument
validation and error types mirror the reference (raster/forward.py:37-41,
raster/backward.py:80-88, raster/backend.py:29-38, camera.py:33-51)."""

import math

import numpy as np
import pytest

from helpers import frontal_view, random_scene, random_view
from paper_2605_18334_b200.camera import CameraView, look_at, to_opencv, world_to_cam, intrinsics
from paper_2605_18334_b200.raster import (MAX_IMAGE_DIM, FrameBundle, FrameMismatchError,
                                          render_backward, render_forward, tile_rect, grid_dims)
from paper_2605_18334_b200.raster.backend import active_backend
from paper_2605_18334_b200.scene import Scene


def test_dimension_overflow_rejected():
    view = CameraView(c2w=np.eye(4), convention="opencv", width=MAX_IMAGE_DIM + 1, height=16,
                      fov_x=0.9)
    with pytest.raises(ValueError):
        render_forward(Scene.empty(), view)


def test_unknown_backend_rejected():
    with pytest.raises(ValueError):
        active_backend("cython")
    with pytest.raises(ValueError):
        render_forward(Scene.empty(), frontal_view(16, 16), backend_name="numpy")
    assert active_backend("cuda") == "cuda"


def test_backend_env(monkeypatch):
    monkeypatch.setenv("SKEWSPLAT_BACKEND", "numpy")
    with pytest.raises(ValueError):
        active_backend()


def _frame(w, h, n, m=0):
    return FrameBundle(color=np.zeros((h, w, 3)), final_T=np.ones((h, w)),
                       n_contrib=np.zeros((h, w), np.int32), last_idx=-np.ones((h, w), np.int64),
                       width=w, height=h, n_primitives=n, n_instances=m, s=0.3)


def test_backward_mismatch_errors_before_device_work():
    rng = np.random.default_rng(1)
    scene = random_scene(rng, 6)
    view = random_view(rng, 32, 32)
    frame = _frame(32, 32, 6)
    dL = np.zeros((32, 32, 3))
    with pytest.raises(FrameMismatchError):
        render_backward(random_scene(rng, 5), view, frame, dL)
    with pytest.raises(FrameMismatchError):
        render_backward(scene, random_view(rng, 16, 32), frame, dL)
    with pytest.raises(FrameMismatchError):
        render_backward(scene, view, frame, np.zeros((16, 16, 3)))
    assert issubclass(FrameMismatchError, ValueError)


def test_camera_conventions_and_intrinsics():
    # reference test_camera.py: T_ALIGN involution, intrinsics, fov_y from aspect
    v = CameraView(np.eye(4), "opengl", 640, 480, 1.0)
    cv = to_opencv(v)
    assert cv.convention == "opencv"
    np.testing.assert_array_equal(cv.c2w, np.diag([1.0, -1.0, -1.0, 1.0]))
    K = intrinsics(CameraView(np.eye(4), "opencv", 640, 480, 1.0))
    assert K[0, 0] == pytest.approx(640 / (2 * math.tan(0.5)))
    assert (K[0, 2], K[1, 2]) == (320.0, 240.0)
    assert v.fov_y == pytest.approx(2 * math.atan(math.tan(0.5) * 480 / 640))
    c2w = look_at([1.0, 2.0, 3.0], [0.0, 0.0, 0.0])
    R, t = world_to_cam(CameraView(c2w, "opencv", 8, 8, 1.0))
    np.testing.assert_allclose(R @ np.array([1.0, 2.0, 3.0]) + t, 0.0, atol=1e-12)
    with pytest.raises(ValueError):
        CameraView(np.eye(4), "dx", 8, 8, 1.0)
    with pytest.raises(ValueError):
        CameraView(np.eye(4), "opencv", 0, 8, 1.0)
    with pytest.raises(ValueError):
        CameraView(np.eye(4), "opencv", 8, 8, 4.0)


def test_scalar_tile_rect_kats():
    # tiles.py:33-40 (host helper); test_raster_forward.py:92-101 rect covers the mean pixel
    ntx, nty = grid_dims(64, 64)
    rng = np.random.default_rng(11)
    for _ in range(100):
        mean = rng.uniform(0.0, 64.0, size=2)
        x0, x1, y0, y1 = tile_rect(mean, rng.uniform(1.0, 5.0), ntx, nty)
        assert x0 <= int(mean[0]) // 16 < x1 and y0 <= int(mean[1]) // 16 < y1


def test_scene_container():
    s = Scene.empty(sh_degree=2)
    assert len(s) == 0 and s.sh.shape == (0, 9, 3)
    with pytest.raises(ValueError):
        Scene(np.zeros((1, 3)), np.zeros((1, 3)), np.zeros((1, 4)), np.zeros((1, 5, 3)),
              np.zeros((1, 2)), np.zeros((1, 3)), np.zeros((1, 3)))
