"""The C ABI library loads on a CPU-only host, exports every function that
include/ssg_b200.h declares, and the ctypes mirrors match the C layouts."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2605_18334_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ssg_b200.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|void|size_t|const char \*)\s*\*?\s*(ssg_\w+)\s*\(", src, re.M)))


def test_header_declares_the_exports():
    assert set(declared_functions()) == set(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = N.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert L.ssg_abi_version() == N.ABI_VERSION


def test_grid_dims_query():
    L = N.lib()
    tx, ty = ctypes.c_int32(), ctypes.c_int32()
    for (w, h), want in (((64, 64), (4, 4)), ((65, 16), (5, 1)), ((1, 1), (1, 1)),
                         ((1920, 1080), (120, 68))):
        L.ssg_grid_dims(w, h, ctypes.byref(tx), ctypes.byref(ty))
        assert (tx.value, ty.value) == want  # tiles.py:29-30, test_raster_forward.py:25-28


def test_ctypes_layouts_match_header(tmp_path):
    structs = {"ssg_scene": N.SsgScene, "ssg_camera": N.SsgCamera, "ssg_params": N.SsgParams,
               "ssg_adam_state": N.SsgAdamState, "ssg_adam_hparams": N.SsgAdamHparams,
               "ssg_prim_buffers": N.SsgPrimBuffers, "ssg_bin_buffers": N.SsgBinBuffers,
               "ssg_frame_buffers": N.SsgFrameBuffers, "ssg_grad_buffers": N.SsgGradBuffers}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append('printf("ssg_splat %zu\\n", sizeof(ssg_splat)); return 0; }')
    c = tmp_path / "layout.c"
    c.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(c)], check=True)
    out = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.split("\n") if l)
    for cname, cls in structs.items():
        assert int(out[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(out[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)
    assert int(out["ssg_splat"]) == N.SPLAT_BYTES


def test_missing_library_fails_loudly(monkeypatch):
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", "/nonexistent/libssg_b200.so")
    with pytest.raises(N.NativeError):
        N.lib()
