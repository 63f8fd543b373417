#!/usr/bin/env bash
# per-kernel durations (ncu, serialised) of one config-2 frame after warm-up
set -u
tag=${1:-ln}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${COUNT:-120} --csv \
  --log-file gpurun_out/${tag}_launches.csv python tools/stage_times.py --reps 2 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/${tag}_launches.csv
