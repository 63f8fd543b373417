#!/usr/bin/env bash
# Builds the UNMODIFIED reference package (Python + its Cython/OpenMP blend
# kernels, raster/_core.pyx) from /root/reference into oracle/_ref/.  The
# build writes into its source tree (cythonize), so it runs on a scratch copy
# under /tmp; only the installed package lands in oracle/_ref/ (git-ignored,
# travels to the GPU box with the snapshot).  /usr/bin/gcc is required: the
# default /opt/gcc lacks libgomp.spec and cannot link -fopenmp.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src=/root/reference/pkg
if [ ! -d "$src" ]; then
  echo "build_ref: $src not present; keeping existing oracle/_ref" >&2
  exit 0
fi
if [ -f "$here/_ref/skewsplat/raster/__init__.py" ] && ls "$here"/_ref/skewsplat/raster/_core*.so >/dev/null 2>&1; then
  exit 0
fi
tmp="$(mktemp -d /tmp/ssg_refbuild.XXXXXX)"
cp -r "$src/." "$tmp/"
rm -rf "$here/_ref"
(cd "$tmp" && CC=/usr/bin/gcc LDSHARED="/usr/bin/gcc -shared" \
   python -m pip install --no-index --no-build-isolation --no-deps -q --target "$here/_ref" .)
rm -rf "$tmp"
