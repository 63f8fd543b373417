#!/usr/bin/env bash
# One GPU session: tests, bench, ncu launch list, ncu full capture of the
# blend kernels.  Outputs under gpurun_out/ (scratch; summaries are copied to
# profiles/ by hand).
set -u
tag=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${tag}_gpu.txt
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_blend -s 6 -c 2 \
  -o gpurun_out/${tag}_blend -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/${tag}_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_preprocess -s 6 -c 2 \
  -o gpurun_out/${tag}_prep -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/${tag}_ncu_prep.log 2>&1
tail -3 gpurun_out/${tag}_pytest.txt; cat gpurun_out/${tag}_bench.json; tail -5 gpurun_out/${tag}_bench.err
