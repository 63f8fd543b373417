"""B200-native rasterizer for 3D Skew Gaussian Splatting (arXiv 2605.18334).

Drop-in for the reference package's rasterizer entry points
(skewsplat.raster.forward.render_forward / backward.render_backward) backed
by hand-written sm_100a CUDA kernels in libssg_b200.so (C ABI:
include/ssg_b200.h).  No CPU fallback exists.
"""

from .camera import OPENCV, OPENGL, CameraView, intrinsics, look_at, to_opencv, world_to_cam
from .ply import PlyError, PlyFormatError, PlyMissingFieldError, PlyTruncatedError, load_ply
from .scene import Scene, SkewGaussian

__all__ = ["CameraView", "Scene", "SkewGaussian", "look_at", "to_opencv", "intrinsics",
           "world_to_cam", "OPENCV", "OPENGL", "load_ply", "PlyError", "PlyFormatError",
           "PlyMissingFieldError", "PlyTruncatedError"]
