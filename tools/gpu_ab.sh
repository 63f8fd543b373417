#!/usr/bin/env bash
# A/B of library variants on the config-2 frame: per-stage device times.
# usage: tools/gpu_ab.sh TAG variant1 variant2 ...   ("base" = libssg_b200.so)
set -u
tag=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2605_18334_b200/libssg_b200.so; else lib=paper_2605_18334_b200/libssg_b200_$v.so; fi
  echo "== $v" >> gpurun_out/${tag}_ab.txt
  SSG_B200_LIB=$lib timeout 300 python tools/stage_times.py --reps 6 2>&1 | tail -3 >> gpurun_out/${tag}_ab.txt
done
cat gpurun_out/${tag}_ab.txt
