#!/usr/bin/env bash
# config-4 bench line per library variant ("base" = libssg_b200.so)
set -u
tag=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2605_18334_b200/libssg_b200.so; else lib=paper_2605_18334_b200/libssg_b200_$v.so; fi
  SSG_B200_LIB=$lib timeout 600 python bench.py --config 4 --steps ${STEPS:-5} --warmup 3 --no-cpu > gpurun_out/${tag}_$v.json 2> gpurun_out/${tag}_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/${tag}_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],3), {k: round(x,4) for k,x in d['stage_ms_per_view'].items()})" >> gpurun_out/${tag}_ab.txt 2>&1
done
cat gpurun_out/${tag}_ab.txt
