"""Rasterizer entry points (drop-in for reference skewsplat.raster)."""

from .backward import FrameMismatchError, GradientBundle, render_backward, screen_gradients
from .forward import MAX_IMAGE_DIM, FrameBundle, render_forward
from .projection import ScreenSplat, project_scene, project_splat
from .tiles import TILE, TileGrid, bin_and_sort, bin_arrays, grid_dims, tile_rect

__all__ = ["render_forward", "render_backward", "screen_gradients", "FrameBundle",
           "GradientBundle", "FrameMismatchError", "MAX_IMAGE_DIM", "TILE", "TileGrid",
           "bin_arrays", "bin_and_sort", "grid_dims", "tile_rect", "ScreenSplat", "project_scene",
           "project_splat"]
