#!/usr/bin/env bash
# ncu --set full of the blend kernels (one frame after warm-up) + hot SASS.
set -u
tag=${1:-nb}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_blend} -s ${SKIP:-6} -c ${COUNT:-2} \
  -o gpurun_out/${tag} -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/${tag}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${tag}.ncu-rep > gpurun_out/${tag}_summary.txt 2>&1
cat gpurun_out/${tag}_summary.txt
