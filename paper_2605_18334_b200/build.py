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
# per-file extra flags: K1 must not contract (tile lists are bit-exact); the
# backward projection recomputes K1's colour clamp and validity, so it rounds
# the same way
EXTRA = {"preprocess_fwd.cu": ["--fmad=false"], "preprocess_bwd.cu": ["--fmad=false"],
         "densify.cu": ["--fmad=false"]}
SOURCES = ["api.cu", "preprocess_fwd.cu", "binning.cu", "blend.cu", "preprocess_bwd.cu", "adam.cu", "train.cu", "densify.cu", "ply.cu", "serve.cu"]
HEADERS = ["ssg_common.cuh", "radix_sort.cuh", "depth_sort.cuh", "onesweep.cuh", "bucket_sort.cuh", os.path.join("..", "..", "include", "ssg_b200.h")]


def _newest_input_mtime(src: str) -> float:
    paths = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS]
    return max(os.path.getmtime(p) for p in paths)


def _compile(src: str, force: bool, obj_dir: str = OBJ_DIR, defines: tuple = ()) -> str:
    obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= _newest_input_mtime(src):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, *defines, *EXTRA.get(src, []), "-c", os.path.join(CSRC, src), "-o", obj]
    subprocess.run(cmd, check=True)
    return obj


def build(force: bool = False, stats: bool = False, variant: str | None = None, defines: tuple = ()) -> str:
    """stats=True builds the diagnostic variant libssg_b200_stats.so (blend
    event counters, tools/blend_stats.py); variant=NAME with extra -D flags
    builds libssg_b200_NAME.so for A/B timing (tools/); neither is ever
    loaded by default."""
    if stats:
        variant, defines = "stats", ("-DSSG_BLEND_STATS",) + tuple(defines)
    obj_dir = OBJ_DIR + (f"_{variant}" if variant else "")
    out = OUT.replace(".so", f"_{variant}.so") if variant else OUT
    defines = tuple(defines)
    os.makedirs(obj_dir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, obj_dir, defines), SOURCES))
    if force or not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "--cudart", "static", "-o", out, *objs]
        subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else None
    print(build(force="--force" in args, stats="--stats" in args, variant=var,
                defines=tuple(a for a in args if a.startswith("-D"))))
