#!/usr/bin/env bash
# per-kernel durations of config-5 training steps (ncu, serialised)
set -u
tag=${1:-c5}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-900} -c ${COUNT:-150} --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --config 5 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu > /dev/null 2>&1
python tools/launch_table.py gpurun_out/${tag}_launches.csv
