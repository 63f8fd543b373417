"""Frame serving on the device: the consumers of the
view-batched forward.

  quantize_u8(img)                      dataset.py:33-38 (one rounding rule
                                        for every output path), on the device
  render_frame(scene, frame_id, view)   service.py:105-107 payload: 8-byte
                                        header (<IHH) + RGB8 pixels; the frame
                                        is quantised on the device, so only
                                        W*H*3 bytes cross PCIe
  render_views_u8(ds, views)            a batch of views -> (V,H,W,3) u8 on
                                        the device (trajectory / service)
  render_trajectory(scene, traj, dir)   trajectory.py:12-31: one PNG per view,
                                        zero-padded names, scene uploaded once
  load_trajectory / save_trajectory     dataset.py camera JSON codec
                                        (trajectory documents)

The WebSocket transport of service.py (FastAPI) is not part of the path.
"""

from __future__ import annotations

import json
import numbers
import os
import struct

import numpy as np
import torch

from . import _native as N
from .camera import OPENCV, OPENGL, CameraView
from .engine import DeviceScene, default_engine, dropin_serialized
from .views import render_views

HEADER = struct.Struct("<IHH")  # service.py:31: frame_id u32, width u16, height u16


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def quantize_u8_device(img: torch.Tensor) -> torch.Tensor:
    """(…,3) f32/f64 device tensor -> u8 device tensor of the same shape."""
    if img.dtype not in (torch.float32, torch.float64) or not img.is_cuda:
        raise ValueError("quantize_u8_device needs a float32/float64 CUDA tensor")
    src = img.contiguous()
    out = torch.empty(src.shape, dtype=torch.uint8, device=src.device)
    N.check(N.lib().ssg_quantize_u8(src.data_ptr(), int(src.dtype == torch.float64), src.numel(), out.data_ptr(),
                                    _stream(src.device)), "ssg_quantize_u8")
    return out


def quantize_u8(img: np.ndarray) -> np.ndarray:
    """dataset.py:33-38 (same validation, same bytes), evaluated on the GPU."""
    arr = np.asarray(img, dtype=np.float64)
    if arr.ndim != 3 or arr.shape[2] != 3:
        raise ValueError("image must be (H, W, 3)")
    dev = default_engine().device
    return quantize_u8_device(torch.from_numpy(np.ascontiguousarray(arr)).to(dev)).cpu().numpy()


def _device_scene(scene, dev) -> DeviceScene:
    if isinstance(scene, DeviceScene):
        return scene
    if isinstance(scene, (str, os.PathLike)):
        from .ply import load_ply_device
        return load_ply_device(scene, dev)
    return DeviceScene.from_host(scene, dev)


@dropin_serialized
def render_frame(scene, frame_id: int, view: CameraView, s: float = 0.3) -> bytes:
    """service.py:105-107: header + RGB8 pixels of `view`."""
    eng = default_engine()
    ds = _device_scene(scene, eng.device)
    f = eng.forward(ds, view, s)
    px = quantize_u8_device(f.color).cpu().numpy()
    return HEADER.pack(frame_id, f.width, f.height) + px.tobytes()


@dropin_serialized
def render_views_u8(scene, views, s: float = 0.3) -> torch.Tensor:
    """Every view of one image size rendered and quantised on the device:
    (V,H,W,3) u8."""
    eng = default_engine()
    ds = _device_scene(scene, eng.device)
    return quantize_u8_device(render_views(ds, views, s, engine=eng))


# -------------------------------------------------- trajectory documents
def _entry_error(index: int, msg: str) -> ValueError:
    return ValueError(f"camera entry {index}: {msg}")


def parse_camera_entry(obj, index: int) -> CameraView:
    """dataset.py:47-75 (trajectory entries: no image file)."""
    if not isinstance(obj, dict):
        raise _entry_error(index, "expected an object")
    for key in ("c2w", "convention", "fov_x", "width", "height"):
        if key not in obj:
            raise _entry_error(index, f"missing field {key!r}")
    c2w = obj["c2w"]
    if not isinstance(c2w, list) or len(c2w) != 16 or not all(isinstance(v, numbers.Real) for v in c2w):
        raise _entry_error(index, "c2w must be a flat list of 16 numbers")
    if obj["convention"] not in (OPENCV, OPENGL):
        raise _entry_error(index, f"unknown convention {obj['convention']!r}")
    try:
        return CameraView(np.asarray(c2w, dtype=np.float64).reshape(4, 4), obj["convention"],
                          int(obj["width"]), int(obj["height"]), float(obj["fov_x"]))
    except (TypeError, ValueError) as e:
        raise _entry_error(index, str(e)) from e


def load_trajectory(path) -> list[CameraView]:
    with open(path, encoding="utf-8") as f:
        doc = json.load(f)
    if not isinstance(doc, list):
        raise ValueError(f"{path}: camera document must be a JSON array")
    return [parse_camera_entry(o, i) for i, o in enumerate(doc)]


def save_trajectory(path, views) -> None:
    doc = [{"c2w": [float(v) for v in np.asarray(view.c2w).reshape(-1)], "convention": view.convention,
            "fov_x": float(view.fov_x), "width": int(view.width), "height": int(view.height)} for view in views]
    with open(path, "w", encoding="utf-8") as f:
        json.dump(doc, f, indent=1)


@dropin_serialized
def render_trajectory(scene, trajectory, out_dir, s: float = 0.3) -> list[str]:
    """trajectory.py:12-31: one PNG per entry, names zero-padded to
    max(4, digits of the last index).  The scene is uploaded once; runs of
    up to 64 consecutive views of one image size render as one device batch
    (views.render_views: one projection pass per 8 views), are quantised on
    the device and come back as one copy, and the PNG encoding -- the
    host-bound part -- runs on a thread pool (zlib releases the GIL) while
    the next batch renders.  Same files, names and bytes as one view at a
    time."""
    from concurrent.futures import ThreadPoolExecutor

    from PIL import Image

    from .views import render_views
    if not isinstance(trajectory, list):
        trajectory = load_trajectory(trajectory)
    os.makedirs(out_dir, exist_ok=True)
    eng = default_engine()
    ds = _device_scene(scene, eng.device)
    width = max(4, len(str(max(len(trajectory) - 1, 0))))
    paths = [os.path.join(out_dir, f"{i:0{width}d}.png") for i in range(len(trajectory))]

    def save(px, path):
        Image.fromarray(px, mode="RGB").save(path, format="PNG")

    with ThreadPoolExecutor(max_workers=max(1, min(8, os.cpu_count() or 1))) as pool:
        pending = []
        i = 0
        while i < len(trajectory):
            size = (int(trajectory[i].width), int(trajectory[i].height))
            j = i + 1
            while (j < len(trajectory) and j - i < 64
                   and (int(trajectory[j].width), int(trajectory[j].height)) == size):
                j += 1
            px = quantize_u8_device(render_views(ds, trajectory[i:j], s, engine=eng)).cpu().numpy()
            pending += [pool.submit(save, px[k], paths[i + k]) for k in range(j - i)]
            i = j
        for fut in pending:
            fut.result()
    return paths
