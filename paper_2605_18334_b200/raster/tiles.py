"""Tile binning (mirror of reference raster/tiles.py:16-96), on the GPU.

`bin_arrays` keeps the reference signature and result type: host fp64
arrays in, TileGrid of int64 numpy arrays out, with instances ordered by
(tile, depth, primitive id) and per-tile half-open ranges equal to
np.searchsorted's.  The work runs in libssg_b200 (ssg_bin_rects +
ssg_bin_prepare + ssg_bin_finish).
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

from ..engine import TILE, default_engine, dropin_serialized, grid_dims  # noqa: F401  (re-exported)


@dataclasses.dataclass
class TileGrid:
    tile_px: int
    tiles_x: int
    tiles_y: int
    ranges: np.ndarray      # (tiles_x*tiles_y, 2) half-open [start, end)
    inst_prim: np.ndarray   # (M,) primitive index per sorted instance
    inst_tile: np.ndarray   # (M,) tile id per sorted instance


def tile_rect(mean2d, radius, tiles_x: int, tiles_y: int):
    """Half-open tile rectangle [x0,x1) x [y0,y1) (tiles.py:33-40); scalar
    helper evaluated on the host, identical arithmetic to the device rect."""
    r = math.ceil(radius)
    x0 = min(tiles_x, max(0, math.floor((mean2d[0] - r) / TILE)))
    x1 = min(tiles_x, max(0, math.floor((mean2d[0] + r) / TILE) + 1))
    y0 = min(tiles_y, max(0, math.floor((mean2d[1] - r) / TILE)))
    y1 = min(tiles_y, max(0, math.floor((mean2d[1] + r) / TILE) + 1))
    return x0, x1, y0, y1


def grid_from_engine(eng, ntx: int, nty: int) -> TileGrid:
    inst_prim, inst_tile, ranges = eng.grid(ntx * nty)
    return TileGrid(TILE, ntx, nty, ranges.cpu().numpy().astype(np.int64),
                    inst_prim.cpu().numpy().astype(np.int64),
                    inst_tile.cpu().numpy().astype(np.int64))


@dropin_serialized
def bin_arrays(mean2d, radius, depth, valid, width: int, height: int) -> TileGrid:
    """Vectorized binning over primitive arrays (tiles.py:43-79)."""
    eng = default_engine()
    dev = eng.device
    mean2d = torch.from_numpy(np.ascontiguousarray(mean2d, dtype=np.float64).reshape(-1, 2)).to(dev)
    n = mean2d.shape[0]
    radius = torch.from_numpy(np.ascontiguousarray(radius, dtype=np.float64).reshape(n)).to(dev)
    depth = torch.from_numpy(np.ascontiguousarray(depth, dtype=np.float64).reshape(n)).to(dev)
    valid = torch.from_numpy(np.ascontiguousarray(valid, dtype=np.uint8).reshape(n)).to(dev)
    eng.bin_arrays(mean2d, radius, depth, valid, int(width), int(height))
    ntx, nty = grid_dims(int(width), int(height))
    return grid_from_engine(eng, ntx, nty)


def bin_and_sort(splats, width: int, height: int) -> TileGrid:
    """List-of-splats variant (tiles.py:82-96): None entries are culled (an
    invalid row), the others binned by their mean, radius and depth."""
    n = len(splats)
    live = [i for i, sp in enumerate(splats) if sp is not None]
    mean2d, radius, depth = np.zeros((n, 2)), np.zeros(n), np.zeros(n)
    valid = np.zeros(n, dtype=bool)
    valid[live] = True
    for i in live:
        mean2d[i], radius[i], depth[i] = splats[i].mean2d, splats[i].radius, splats[i].depth
    return bin_arrays(mean2d, radius, depth, valid, width, height)
