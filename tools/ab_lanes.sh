#!/usr/bin/env bash
# config-4 bench line for several view-lane counts
set -u
tag=$1; shift
mkdir -p gpurun_out
for l in "$@"; do
  timeout 600 python bench.py --config 4 --steps ${STEPS:-5} --warmup 3 --no-cpu --lanes $l > gpurun_out/${tag}_l$l.json 2> gpurun_out/${tag}_l$l.err
  python -c "
import json; d=json.loads(open('gpurun_out/${tag}_l$l.json').read().strip().splitlines()[-1]); print('lanes $l', round(d['value'],1), round(d['ms_per_step'],3))" >> gpurun_out/${tag}_ab.txt 2>&1
  tail -2 gpurun_out/${tag}_l$l.err >> gpurun_out/${tag}_ab.txt
done
cat gpurun_out/${tag}_ab.txt
