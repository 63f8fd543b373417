#!/usr/bin/env bash
# view-batch tests + the config-4 bench line (+ optional ncu of the batched projection)
set -u
tag=${1:-c4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_view_batch.py tests/test_gpu_configs.py tests/test_gpu_syncfree.py -x -q > gpurun_out/${tag}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 900 python bench.py --config 4 --steps ${STEPS:-5} --warmup 3 --no-cpu > gpurun_out/${tag}_c4.json 2> gpurun_out/${tag}_c4.err
if [ -n "${NCU:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_preprocess_forward_views" -s 8 -c 1 \
    -o gpurun_out/${tag}_pfv -f python bench.py --config 4 --steps 1 --warmup 3 --no-cpu > gpurun_out/${tag}_ncu_pfv.log 2>&1
  python tools/ncu_stalls.py gpurun_out/${tag}_pfv.ncu-rep > gpurun_out/${tag}_stalls_pfv.txt 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_pfv.ncu-rep > gpurun_out/${tag}_ncu_pfv.txt 2>&1
fi
tail -5 gpurun_out/${tag}_pytest.txt; python -c "
import json,sys; d=json.loads(open('gpurun_out/${tag}_c4.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['stage_ms_per_view'])"; tail -3 gpurun_out/${tag}_c4.err
cat gpurun_out/${tag}_stalls_pfv.txt 2>/dev/null
