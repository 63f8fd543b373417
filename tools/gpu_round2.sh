#!/usr/bin/env bash
# One GPU session (round 2): tests, full-size parity, bench lines of configs 2-5,
# the ncu launch list, ncu --set full of the blend / preprocess / binning kernels
# and their stall + pipe breakdown.  Outputs under gpurun_out/ (scratch).
set -u
tag=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${tag}_gpu.txt
nproc >> gpurun_out/${tag}_gpu.txt
if [ -z "${NO_TESTS:-}" ]; then
  timeout 1800 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/${tag}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
fi
if [ -z "${NO_PARITY:-}" ]; then
  timeout 1200 python tools/parity_at_scale.py c2 c4 > gpurun_out/${tag}_parity.jsonl 2> gpurun_out/${tag}_parity.err
fi
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
for c in 3 4 5; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu > gpurun_out/${tag}_c$c.json 2> gpurun_out/${tag}_c$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu > /dev/null 2>&1
python tools/launch_table.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launch_table.txt 2>&1
if [ -z "${NO_NCU:-}" ]; then
for k in blend preprocess sort cs; do
  case $k in blend) rx="k_blend"; sk=6; c=2;; preprocess) rx="k_preprocess"; sk=6; c=2;;
             sort) rx="k_count|k_scan|k_scatter|k_rank|k_minmax|k_depth_sort"; sk=0; c=8;; cs) rx="k_cs"; sk=24; c=8;; esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $sk -c $c \
    -o gpurun_out/${tag}_$k -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/${tag}_ncu_$k.log 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_$k.ncu-rep > gpurun_out/${tag}_ncu_$k.txt 2>&1
  python tools/ncu_stalls.py gpurun_out/${tag}_$k.ncu-rep > gpurun_out/${tag}_stalls_$k.txt 2>&1
done
fi
tail -15 gpurun_out/${tag}_pytest.txt 2>/dev/null; cat gpurun_out/${tag}_bench.json; tail -5 gpurun_out/${tag}_bench.err; head -30 gpurun_out/${tag}_launch_table.txt
