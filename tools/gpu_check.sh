#!/usr/bin/env bash
# GPU round check: tests, full-size parity, one bench line.  usage: tools/gpu_check.sh TAG [pytest-args]
set -u
tag=${1:-chk}; shift || true
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${@:-} > gpurun_out/${tag}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 900 python tools/parity_at_scale.py c2 c4 > gpurun_out/${tag}_parity.jsonl 2> gpurun_out/${tag}_parity.err
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -15 gpurun_out/${tag}_pytest.txt; tail -3 gpurun_out/${tag}_bench.err
