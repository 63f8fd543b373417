"""Scene PLY I/O against the reference's own
save_ply / load_ply (oracle/_ref): identical bytes written, identical scenes
read, the same errors; plus the device unpack (GPU)."""

import os
import sys

import numpy as np
import pytest

from helpers import random_scene
from paper_2605_18334_b200.ply import (PlyFormatError, PlyMissingFieldError, PlyTruncatedError, load_ply,
                                       load_ply_device, save_ply)
from paper_2605_18334_b200.scene import Scene

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = Scene.ARRAY_FIELDS


def _ref():
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "skewsplat")):
        pytest.skip("oracle/_ref not present")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import skewsplat.scene as S
    return S


def _same(a, b):
    assert a.sh_degree == b.sh_degree and len(a) == len(b)
    np.testing.assert_array_equal(a.background, b.background)
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)


def _standard_3dgs(path, n=5, degree=1, seed=4, types=None, drop=None, truncate=0, fmt="binary_little_endian"):
    """A plain-Gaussian export with per-property types (mixed widths make
    the record stride unaligned)."""
    rng = np.random.default_rng(seed)
    m = (degree + 1) ** 2 - 1
    names = (["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"] + [f"f_rest_{i}" for i in range(3 * m)]
             + ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"])
    if drop:
        names = [nm for nm in names if nm != drop]
    types = types or {}
    tmap = {"<f4": "float", "<f8": "double", "<u1": "uchar", "<i2": "short", "<u2": "ushort", "<i4": "int",
            "<u4": "uint", "<i1": "char"}
    dts = [(nm, types.get(nm, "<f4")) for nm in names]
    data = np.zeros(n, dtype=dts)
    for nm, t in dts:
        v = rng.normal(size=n) * (3 if np.dtype(t).kind == "f" else 40)
        data[nm] = np.abs(v) if np.dtype(t).kind == "u" else v
    lines = ["ply", f"format {fmt} 1.0", f"element vertex {n}"] + [f"property {tmap[t]} {nm}" for nm, t in dts]
    lines.append("end_header")
    blob = ("\n".join(lines) + "\n").encode() + data.tobytes()
    if truncate:
        blob = blob[:-truncate]
    path.write_bytes(blob)


def test_save_is_byte_identical_and_round_trips(tmp_path):
    S = _ref()
    rng = np.random.default_rng(3)
    ours = random_scene(rng, 17, sh_degree=2)
    theirs = S.Scene(*(getattr(ours, f).copy() for f in FIELDS), background=ours.background.copy(),
                     sh_degree=ours.sh_degree)
    save_ply(ours, tmp_path / "a.ply")
    theirs.save_ply(tmp_path / "b.ply")
    assert (tmp_path / "a.ply").read_bytes() == (tmp_path / "b.ply").read_bytes()
    _same(load_ply(tmp_path / "a.ply"), ours)
    _same(load_ply(tmp_path / "b.ply"), S.load_ply(tmp_path / "b.ply"))


def test_empty_scene(tmp_path):
    scene = Scene.empty(sh_degree=1, background=(0.25, 0.5, 0.75))
    scene.save_ply(tmp_path / "e.ply")
    back = load_ply(tmp_path / "e.ply")
    assert len(back) == 0 and back.sh_degree == 1
    np.testing.assert_array_equal(back.background, [0.25, 0.5, 0.75])


@pytest.mark.parametrize("degree", [0, 1, 3])
def test_standard_3dgs_import_matches_reference(tmp_path, degree):
    S = _ref()
    p = tmp_path / "plain.ply"
    _standard_3dgs(p, n=9, degree=degree, types={"x": "<f8", "opacity": "<i2", "rot_1": "<u1"})
    _same(load_ply(p), S.load_ply(p))


@pytest.mark.parametrize("kw,err,match", [({"drop": "opacity"}, PlyMissingFieldError, "opacity"),
                                          ({"truncate": 7}, PlyTruncatedError, None),
                                          ({"fmt": "ascii"}, PlyFormatError, "ascii")])
def test_errors_match_reference(tmp_path, kw, err, match):
    S = _ref()
    p = tmp_path / "bad.ply"
    _standard_3dgs(p, **kw)
    with pytest.raises(err, match=match):
        load_ply(p)
    with pytest.raises(ValueError):
        S.load_ply(p)
    (tmp_path / "junk.ply").write_bytes(b"\x89PNG not a ply")
    with pytest.raises(PlyFormatError):
        load_ply(tmp_path / "junk.ply")


@pytest.mark.gpu
@pytest.mark.parametrize("types", [None, {"x": "<f8", "opacity": "<i2", "rot_1": "<u1", "f_dc_2": "<u2"}])
def test_device_unpack_equals_host_load(tmp_path, types):
    import torch
    from paper_2605_18334_b200.engine import DeviceScene
    p = tmp_path / "s.ply"
    _standard_3dgs(p, n=3001, degree=3, types=types)
    host = DeviceScene.from_host(load_ply(p))
    dev = load_ply_device(p)
    assert dev.n == host.n and dev.sh_degree == host.sh_degree
    for f in ("mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir"):
        assert torch.equal(getattr(dev, f), getattr(host, f)), f
    rng = np.random.default_rng(1)
    scene = random_scene(rng, 500, sh_degree=2)
    scene.save_ply(tmp_path / "r.ply")
    host, dev = DeviceScene.from_host(scene), load_ply_device(tmp_path / "r.ply")
    for f in ("mu", "log_scale", "rot", "sh", "opacity_logits", "beta", "dir"):
        assert torch.equal(getattr(dev, f), getattr(host, f)), f
