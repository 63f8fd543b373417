"""Scene PLY I/O.

Same file format and behaviour as the reference (scene.py:168-313): binary
little-endian, one `vertex` element, properties read by name, SH rest
coefficients channel-major, `comment background` / `comment sh_degree`
header comments, the same error classes and messages' meaning.

  load_ply(path) -> Scene                  host, numpy (the reference's API)
  save_ply(scene, path)                    byte-identical output to Scene.save_ply
  load_ply_device(path) -> DeviceScene     header parsed on the host, the raw
                                           vertex payload uploaded once and
                                           unpacked into the device SoA layout by
                                           the ssg_ply_unpack kernel
"""

from __future__ import annotations

import ctypes
import io
import math

import numpy as np

from .scene import Scene

PLY_TYPES = {  # scene.py:210-216
    "float": ("<f4", 0), "float32": ("<f4", 0),
    "double": ("<f8", 1), "float64": ("<f8", 1),
    "char": ("<i1", 2), "int8": ("<i1", 2), "uchar": ("<u1", 3), "uint8": ("<u1", 3),
    "short": ("<i2", 4), "int16": ("<i2", 4), "ushort": ("<u2", 5), "uint16": ("<u2", 5),
    "int": ("<i4", 6), "int32": ("<i4", 6), "uint": ("<u4", 7), "uint32": ("<u4", 7),
}
REQUIRED = ("x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
            "rot_0", "rot_1", "rot_2", "rot_3")


class PlyError(ValueError):
    """Base class for PLY parsing failures (scene.py:23-24)."""


class PlyFormatError(PlyError):
    pass


class PlyMissingFieldError(PlyError):
    def __init__(self, field: str):
        super().__init__(f"missing mandatory vertex property: {field}")
        self.field = field


class PlyTruncatedError(PlyError):
    def __init__(self, expected: int, got: int):
        super().__init__(f"truncated payload: expected {expected} bytes, got {got}")
        self.expected, self.got = expected, got


class PlyHeader:
    """Parsed header: vertex count, property layout, background, SH degree."""

    def __init__(self, raw: bytes):
        marker = b"end_header\n"
        end = raw.find(marker)
        if not raw.startswith(b"ply\n") or end < 0:
            raise PlyFormatError("not a PLY file (missing ply/end_header)")
        lines = raw[:end].decode("ascii", errors="replace").splitlines()
        self.payload_offset = end + len(marker)
        fmt = [ln for ln in lines if ln.startswith("format ")]
        if not fmt:
            raise PlyFormatError("missing format line")
        if "binary_little_endian" not in fmt[0]:
            raise PlyFormatError(f"unsupported format: {fmt[0].split()[1]}")
        self.background = np.zeros(3)
        hint = None
        for ln in lines:
            if ln.startswith("comment background "):
                self.background = np.array([float(v) for v in ln.split()[2:5]])
            elif ln.startswith("comment sh_degree "):
                hint = int(ln.split()[2])
        self.n = None
        self.props: list[tuple[str, str, int]] = []  # name, numpy type, ssg type code
        in_vertex = False
        for ln in lines:
            tok = ln.split()
            if not tok:
                continue
            if tok[0] == "element":
                in_vertex = tok[1] == "vertex"
                if in_vertex:
                    self.n = int(tok[2])
            elif tok[0] == "property" and in_vertex:
                if tok[1] == "list":
                    raise PlyFormatError("list properties are not supported on vertices")
                if tok[1] not in PLY_TYPES:
                    raise PlyFormatError(f"unsupported property type: {tok[1]}")
                np_t, code = PLY_TYPES[tok[1]]
                self.props.append((tok[2], np_t, code))
        if self.n is None:
            raise PlyFormatError("missing 'element vertex' declaration")
        self.names = [p[0] for p in self.props]
        for f in REQUIRED:
            if f not in self.names:
                raise PlyMissingFieldError(f)
        self.dtype = np.dtype([(nm, t) for nm, t, _ in self.props])
        n_rest = sum(nm.startswith("f_rest_") for nm in self.names)
        if n_rest % 3:
            raise PlyFormatError(f"f_rest_* count {n_rest} is not a multiple of 3")
        self.m = n_rest // 3
        deg = int(round(math.sqrt(self.m + 1))) - 1
        if (deg + 1) ** 2 - 1 != self.m or deg > 3:
            raise PlyFormatError(f"f_rest_* count {n_rest} does not match any SH degree <= 3")
        if hint is not None and hint != deg:
            raise PlyFormatError(f"header sh_degree {hint} contradicts f_rest_* count {n_rest}")
        self.sh_degree = deg
        self.K = (deg + 1) ** 2

    def check_payload(self, nbytes: int):
        need = self.n * self.dtype.itemsize
        if nbytes < need:
            raise PlyTruncatedError(need, nbytes)
        return need

    def component_sources(self) -> list[str | None]:
        """Property name feeding each destination component of ssg_ply_unpack
        (mu, log_scale, rot, logits, beta, dir, sh coefficient-major then RGB);
        None = absent (0)."""
        have = set(self.names)
        opt3 = lambda stem: [f"{stem}_{i}" if f"{stem}_0" in have else None for i in range(3)]  # noqa: E731
        src = ["x", "y", "z"] + [f"scale_{i}" for i in range(3)] + [f"rot_{i}" for i in range(4)]
        src += ["opacity", "opacity2" if "opacity2" in have else "opacity"]  # scene.py:297-298
        src += opt3("skew") + opt3("dir")
        for k in range(self.K):
            for c in range(3):
                src.append(f"f_dc_{c}" if k == 0 else f"f_rest_{c * self.m + k - 1}")
        return src


def _read(path) -> tuple[PlyHeader, bytes]:
    with open(path, "rb") as f:
        raw = f.read()
    return PlyHeader(raw), raw


def load_ply(path) -> Scene:
    """scene.py:222-313 on the host: every column converted to fp64."""
    h, raw = _read(path)
    payload = memoryview(raw)[h.payload_offset:]
    need = h.check_payload(len(payload))
    data = np.frombuffer(payload[:need], dtype=h.dtype)
    src = h.component_sources()
    cols = [np.zeros(h.n) if s is None else np.asarray(data[s], dtype=np.float64) for s in src]
    st = lambda a, b: np.stack(cols[a:b], axis=1)  # noqa: E731
    sh = np.stack(cols[18:], axis=1).reshape(h.n, h.K, 3)
    return Scene(st(0, 3), st(3, 6), st(6, 10), sh, st(10, 12), st(12, 15), st(15, 18),
                 background=h.background, sh_degree=h.sh_degree)


def vertex_names(sh_coeffs: int) -> list[str]:
    """scene.py:168-175 property order."""
    n_rest = (sh_coeffs - 1) * 3
    return (["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2"] + [f"f_rest_{i}" for i in range(n_rest)] +
            ["opacity", "opacity2", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3",
             "skew_0", "skew_1", "skew_2", "dir_0", "dir_1", "dir_2"])


def save_ply(scene, path):
    """scene.py:177-207: fp64 properties, rest coefficients channel-major."""
    n, K = len(scene.mu), scene.sh.shape[1]
    names = vertex_names(K)
    rec = np.empty(n, dtype=[(nm, "<f8") for nm in names])
    rec["x"], rec["y"], rec["z"] = scene.mu[:, 0], scene.mu[:, 1], scene.mu[:, 2]
    for c in range(3):
        rec[f"f_dc_{c}"] = scene.sh[:, 0, c]
        for j in range(K - 1):
            rec[f"f_rest_{c * (K - 1) + j}"] = scene.sh[:, 1 + j, c]
    rec["opacity"], rec["opacity2"] = scene.opacity_logits[:, 0], scene.opacity_logits[:, 1]
    for i in range(3):
        rec[f"scale_{i}"] = scene.log_scale[:, i]
        rec[f"skew_{i}"] = scene.beta[:, i]
        rec[f"dir_{i}"] = scene.dir[:, i]
    for i in range(4):
        rec[f"rot_{i}"] = scene.rot[:, i]
    hdr = io.StringIO()
    hdr.write("ply\nformat binary_little_endian 1.0\n")
    hdr.write("comment background " + " ".join("%.17g" % v for v in np.asarray(scene.background)) + "\n")
    hdr.write(f"comment sh_degree {scene.sh_degree}\nelement vertex {n}\n")
    for nm in names:
        hdr.write(f"property double {nm}\n")
    hdr.write("end_header\n")
    with open(path, "wb") as f:
        f.write(hdr.getvalue().encode("ascii"))
        f.write(rec.tobytes())


def load_ply_device(path, device=None):
    """PLY -> DeviceScene: host header parse, one upload of the raw vertex
    payload, device unpack (ssg_ply_unpack) into the SoA scene layout."""
    import torch

    from . import _native as N
    from .engine import DeviceScene
    h, raw = _read(path)
    need = h.check_payload(len(raw) - h.payload_offset)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n, K = h.n, h.K
    offs = {nm: h.dtype.fields[nm][1] for nm in h.names}
    code = {nm: c for nm, _, c in h.props}
    src = h.component_sources()
    off_arr = (ctypes.c_int32 * len(src))(*[offs[s] if s else 0 for s in src])
    typ_arr = (ctypes.c_int32 * len(src))(*[code[s] if s else -1 for s in src])
    m = max(n, 1)
    ds = DeviceScene(torch.empty((m, 3), dtype=torch.float64, device=dev)[:n],
                     torch.empty((m, 3), dtype=torch.float64, device=dev)[:n],
                     torch.empty((m, 4), dtype=torch.float64, device=dev)[:n],
                     torch.empty((m, K, 3), dtype=torch.float32, device=dev)[:n],
                     torch.empty((m, 2), dtype=torch.float32, device=dev)[:n],
                     torch.empty((m, 3), dtype=torch.float32, device=dev)[:n],
                     torch.empty((m, 3), dtype=torch.float32, device=dev)[:n], h.background, h.sh_degree)
    if n:
        payload = torch.frombuffer(bytearray(raw[h.payload_offset:h.payload_offset + need]), dtype=torch.uint8)
        payload = payload.pin_memory().to(dev, non_blocking=True)
        p = N.SsgParams()
        p.n, p.sh_degree, p.sh_coeffs = n, h.sh_degree, K
        for f in ("mu", "log_scale", "rot", "sh", "beta", "dir"):
            setattr(p, f, getattr(ds, f).data_ptr())
        p.opacity_logits = ds.opacity_logits.data_ptr()
        N.check(N.lib().ssg_ply_unpack(payload.data_ptr(), n, h.dtype.itemsize, off_arr, typ_arr, K,
                                       ctypes.byref(p), torch.cuda.current_stream(dev).cuda_stream),
                "ssg_ply_unpack")
        torch.cuda.current_stream(dev).synchronize()
    return ds
