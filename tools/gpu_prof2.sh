#!/usr/bin/env bash
# launch list of the config-4 frame (ball scene, view 0) and ncu --set full of
# the config-2 forward blend + exact paths and the config-4 binning kernels
set -u
tag=${1:-p2}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/${tag}_c4_launches.csv python tools/stage_times.py --ball --reps 2 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/${tag}_c4_launches.csv > gpurun_out/${tag}_c4_launch_table.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_blend_forward" -s 3 -c 3 \
  -o gpurun_out/${tag}_fwd -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/${tag}_ncu_fwd.log 2>&1
python tools/ncu_stalls.py gpurun_out/${tag}_fwd.ncu-rep > gpurun_out/${tag}_stalls_fwd.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pass|k_hist|k_minmax|k_fixup|k_count_scan|k_cs" -s 14 -c 14 \
  -o gpurun_out/${tag}_c4bin -f python tools/stage_times.py --ball --reps 1 > gpurun_out/${tag}_ncu_c4bin.log 2>&1
python tools/ncu_stalls.py gpurun_out/${tag}_c4bin.ncu-rep > gpurun_out/${tag}_stalls_c4bin.txt 2>&1
cat gpurun_out/${tag}_c4_launch_table.txt | head -40; cat gpurun_out/${tag}_stalls_fwd.txt gpurun_out/${tag}_stalls_c4bin.txt
