# sort tests + binning parity + per-kernel launch list of the binning (c2, c4)
mkdir -p gpurun_out
tag=${1:-r2z}
timeout 600 python -m pytest tests/test_gpu_sort.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q > gpurun_out/${tag}_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 300 python tools/stage_times.py --reps 6 2>&1 | tail -2 | head -1 > gpurun_out/${tag}_stages.txt
timeout 300 python tools/stage_times.py --reps 6 --ball 2>&1 | tail -2 | head -1 >> gpurun_out/${tag}_stages.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_c2.csv python tools/stage_times.py --reps 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_c4.csv python tools/stage_times.py --reps 2 --ball > /dev/null 2>&1
tail -3 gpurun_out/${tag}_pytest.txt; cat gpurun_out/${tag}_stages.txt
