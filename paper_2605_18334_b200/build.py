"""Build libssg_b200.so in-tree with nvcc for sm_100a.

Usage: python -m paper_2605_18334_b200.build [--force]
The shared library lands next to this file so it travels with the repo
snapshot to the GPU box (no JIT cache under ~/.cache).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libssg_b200.so")
OBJ_DIR = os.path.join(HERE, "csrc", "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
# per-file extra flags: K1 must not contract (tile lists are bit-exact)
EXTRA = {"preprocess_fwd.cu": ["--fmad=false"]}
SOURCES = ["api.cu", "preprocess_fwd.cu", "binning.cu", "blend.cu", "preprocess_bwd.cu", "adam.cu"]
HEADERS = ["ssg_common.cuh", "radix_sort.cuh", os.path.join("..", "..", "include", "ssg_b200.h")]


def _newest_input_mtime(src: str) -> float:
    paths = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS]
    return max(os.path.getmtime(p) for p in paths)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ_DIR, src.replace(".cu", ".o"))
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= _newest_input_mtime(src):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, *EXTRA.get(src, []), "-c", os.path.join(CSRC, src), "-o", obj]
    subprocess.run(cmd, check=True)
    return obj


def build(force: bool = False) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), SOURCES))
    if force or not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "--cudart", "static", "-o", OUT, *objs]
        subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
