#!/usr/bin/env bash
# One GPU session: tests, bench, ncu launch list, ncu full captures of the
# blend, preprocess and binning kernels.  Outputs under gpurun_out/ (scratch;
# summaries are copied to profiles/ by hand).
set -u
tag=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${tag}_gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu > /dev/null 2>&1
python tools/launch_table.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launch_table.txt 2>&1
# skip the warm-up frames: 3 warm-up + 2 timed frames of the value loop come first
for k in blend preprocess depth_sort cs; do
  case $k in blend) rx="k_blend"; sk=6; c=2;; preprocess) rx="k_preprocess"; sk=6; c=2;;
             depth_sort) rx="k_depth_sort"; sk=3; c=1;; cs) rx="k_cs"; sk=24; c=8;; esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $sk -c $c \
    -o gpurun_out/${tag}_$k -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/${tag}_ncu_$k.log 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_$k.ncu-rep > gpurun_out/${tag}_ncu_$k.txt 2>&1
done
tail -3 gpurun_out/${tag}_pytest.txt; cat gpurun_out/${tag}_bench.json; tail -5 gpurun_out/${tag}_bench.err; cat gpurun_out/${tag}_launch_table.txt | head -24
