#!/usr/bin/env bash
# A/B stage timings of library variants on config 2:
#   bash tools/ab_blend.sh tag name1 name2 ...   (libssg_b200_<name>.so; "main" = default build)
set -u
tag=$1; shift
mkdir -p gpurun_out
out=gpurun_out/${tag}_ab.txt; : > $out
for v in "$@"; do
  lib=paper_2605_18334_b200/libssg_b200_${v}.so; [ "$v" = main ] && lib=paper_2605_18334_b200/libssg_b200.so
  echo "== $v" >> $out
  SSG_B200_LIB=$lib timeout 300 python tools/stage_times.py --reps 6 ${STAGE_ARGS:-} 2>&1 | tail -3 >> $out
done
cat $out
