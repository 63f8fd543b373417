"""The reference's projection / binning helpers on the device path:
project_splat and ScreenSplat (projection.py:29-38, 238-252; reference
test_projection.py:226-245), bin_and_sort and bin_arrays (tiles.py:43-96;
reference test_raster_forward.py:24-101)."""

import math

import numpy as np
import pytest

from helpers import frontal_view, single_splat_scene
from oracle import oracle as O
from paper_2605_18334_b200.raster import bin_and_sort, bin_arrays, grid_dims, project_scene, project_splat
from paper_2605_18334_b200.scene import Scene

pytestmark = pytest.mark.gpu


def center_fixture():
    view = frontal_view(64, 64)
    g = single_splat_scene((32.0, 32.0), view, 0.5, (1.0, 0.2, 0.1), beta=np.array([0.3, -0.2, 0.1]),
                           direc=np.array([0.1, 0.1, 0.0]))
    return Scene.from_primitives([g]), view, g


def test_project_splat_behind_camera_returns_none():
    _, view, g = center_fixture()
    g.mu = np.array([0.0, 0.0, -1.0])
    assert project_splat(g, view) is None


def test_project_splat_far_offscreen_returns_none():
    _, view, g = center_fixture()
    g.mu = np.array([500.0, 0.0, 5.0])
    assert project_splat(g, view) is None


def test_project_splat_fields_match_vectorized_path_and_oracle():
    scene, view, g = center_fixture()
    sp = project_splat(g, view, s=0.3)
    p = project_scene(scene, view, s=0.3)
    np.testing.assert_array_equal(sp.mean2d, p.mean2d[0])
    assert (sp.conic.a, sp.conic.b, sp.conic.c) == tuple(p.conic[0])
    assert (sp.skew2d.beta_x, sp.skew2d.beta_y) == tuple(p.skew2d[0])
    assert sp.depth == p.depth[0] and sp.dilation_comp == p.comp[0] and sp.radius == p.radius[0]
    ref = O.project(scene, view, 0.3)
    np.testing.assert_array_equal(p.mean2d, ref.mean2d)
    np.testing.assert_array_equal(p.depth, ref.depth)
    # the skew factor is v / sqrt(1 + p - u.v): the cancellation in p - u.v
    # turns last-bit differences (device FMA contraction) into ~1e-8 relative
    for got, want, tol in ((p.conic, ref.conic, 1e-12), (p.skew2d, ref.skew2d, 1e-6),
                           (p.opacity_pair, ref.opacity_pair, 1e-12), (p.comp, ref.comp, 1e-12),
                           (p.radius, ref.radius, 1e-12)):
        np.testing.assert_allclose(got, want, rtol=tol, atol=1e-300)
    np.testing.assert_allclose(p.color, ref.color, rtol=1e-5, atol=1e-6)


def _bin_single(mean, radius, depth, w, h):
    return bin_arrays(np.array([mean]), np.array([radius]), np.array([depth]), np.array([True]), w, h)


def test_binning_cases():
    assert grid_dims(64, 64) == (4, 4) and grid_dims(65, 16) == (5, 1) and grid_dims(1, 1) == (1, 1)
    grid = bin_and_sort([], 64, 48)
    assert grid.ranges.shape == (12, 2) and np.all(grid.ranges == 0) and grid.inst_prim.size == 0
    grid = _bin_single((24.0, 24.0), 3.0, 5.0, 64, 64)
    tid = 1 * grid.tiles_x + 1
    assert grid.inst_prim.tolist() == [0] and grid.inst_tile.tolist() == [tid]
    assert grid.ranges[tid].tolist() == [0, 1]
    grid = _bin_single((30.0, 8.0), 4.0, 5.0, 64, 64)
    assert grid.inst_prim.size == 2 and sorted(grid.inst_tile.tolist()) == [1, 2]
    mean, rad = np.array([[8.0, 8.0], [9.0, 9.0]]), np.array([2.0, 2.0])
    assert bin_arrays(mean, rad, np.array([5.0, 2.0]), np.array([True, True]), 32, 32).inst_prim.tolist() == [1, 0]
    assert bin_arrays(mean, rad, np.array([3.0, 3.0]), np.array([True, True]), 32, 32).inst_prim.tolist() == [0, 1]
    assert bin_arrays(mean, rad, np.array([1.0, 2.0]), np.array([False, True]), 32, 32).inst_prim.tolist() == [1]
    assert bin_and_sort([None, None], 32, 32).inst_prim.size == 0
    assert _bin_single((-100.0, -100.0), 3.0, 5.0, 64, 64).inst_prim.size == 0
    assert _bin_single((500.0, 30.0), 3.0, 5.0, 64, 64).inst_prim.size == 0


def test_bin_and_sort_of_projected_splats_equals_bin_arrays():
    rng = np.random.default_rng(4)
    view = frontal_view(96, 64)
    prims = [single_splat_scene((float(x), float(y)), view, 0.6, (0.5, 0.5, 0.5), scale=0.05 + 0.1 * u,
                                depth=3.0 + 5.0 * u)
             for x, y, u in zip(rng.uniform(-20, 116, 40), rng.uniform(-20, 84, 40), rng.uniform(0, 1, 40))]
    splats = [project_splat(g, view) for g in prims]
    assert any(sp is None for sp in splats) and any(sp is not None for sp in splats)
    grid = bin_and_sort(splats, 96, 64)
    p = project_scene(Scene.from_primitives(prims), view)
    onscreen = np.array([sp is not None for sp in splats])
    ref = O.bin_arrays(p.mean2d, p.radius, p.depth, p.valid & onscreen, 96, 64)
    np.testing.assert_array_equal(grid.inst_prim, ref.inst_prim)
    np.testing.assert_array_equal(grid.ranges, ref.ranges)
    assert math.isfinite(float(p.radius.sum()))
