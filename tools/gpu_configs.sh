#!/usr/bin/env bash
# bench lines of configs 3, 4, 5 (config 2 is the default bench)
set -u
tag=${1:-cfg}
mkdir -p gpurun_out
for c in 3 4 5; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 > gpurun_out/${tag}_c$c.json 2> gpurun_out/${tag}_c$c.err
  tail -c 1500 gpurun_out/${tag}_c$c.json; tail -3 gpurun_out/${tag}_c$c.err
done
