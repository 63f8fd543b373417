#!/usr/bin/env bash
# tile sort vs the counting scatter: binning-related tests, then stage times (configs 2 and 4)
set -u
tag=${1:-ts}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_edges.py tests/test_gpu_syncfree.py tests/test_gpu_exact.py tests/test_gpu_view_batch.py -x -q > gpurun_out/${tag}_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.txt
for v in ${VARIANTS:-base cs}; do
  if [ "$v" = base ]; then lib=paper_2605_18334_b200/libssg_b200.so; else lib=paper_2605_18334_b200/libssg_b200_$v.so; fi
  echo "== $v c2" >> gpurun_out/${tag}_ab.txt
  SSG_B200_LIB=$lib timeout 300 python tools/stage_times.py --reps 6 2>&1 | tail -2 | head -1 >> gpurun_out/${tag}_ab.txt
  echo "== $v c4" >> gpurun_out/${tag}_ab.txt
  SSG_B200_LIB=$lib timeout 300 python tools/stage_times.py --reps 6 --ball 2>&1 | tail -2 | head -1 >> gpurun_out/${tag}_ab.txt
done
if [ -n "${LAUNCHES:-}" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/${tag}_c4_launches.csv python tools/stage_times.py --ball --reps 2 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/${tag}_c4_launches.csv > gpurun_out/${tag}_c4_launch_table.txt 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/${tag}_c2_launches.csv python tools/stage_times.py --reps 2 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/${tag}_c2_launches.csv > gpurun_out/${tag}_c2_launch_table.txt 2>&1
fi
tail -15 gpurun_out/${tag}_pytest.txt; cat gpurun_out/${tag}_ab.txt; tail -32 gpurun_out/${tag}_c4_launch_table.txt 2>/dev/null; tail -32 gpurun_out/${tag}_c2_launch_table.txt 2>/dev/null
