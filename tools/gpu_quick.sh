#!/usr/bin/env bash
# Quick GPU check: GPU tests, one bench line, blend event counters.
set -u
tag=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
if [ -f paper_2605_18334_b200/libssg_b200_stats.so ]; then
  SSG_B200_LIB=paper_2605_18334_b200/libssg_b200_stats.so timeout 300 python tools/blend_stats.py > gpurun_out/${tag}_stats.txt 2>&1
fi
tail -5 gpurun_out/${tag}_pytest.txt; cat gpurun_out/${tag}_bench.json; tail -3 gpurun_out/${tag}_bench.err; cat gpurun_out/${tag}_stats.txt 2>/dev/null
