#!/usr/bin/env bash
set -u
tag=${1:-nt}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"${KREGEX:-tsort::}" -s ${SKIP:-8} -c ${COUNT:-8} \
  -o gpurun_out/${tag} -f python tools/stage_times.py --reps 2 > gpurun_out/${tag}_ncu.log 2>&1
python tools/ncu_stalls.py gpurun_out/${tag}.ncu-rep > gpurun_out/${tag}_stalls.txt 2>&1
python tools/ncu_summary.py gpurun_out/${tag}.ncu-rep > gpurun_out/${tag}_summary.txt 2>&1
cat gpurun_out/${tag}_stalls.txt; grep -i "dram__bytes\|L2 Hit\|DRAM Through" gpurun_out/${tag}_summary.txt
