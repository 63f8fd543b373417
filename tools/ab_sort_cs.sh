mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sort.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q > gpurun_out/r2x_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2x_pytest.txt
for v in base os1 csa csb csc csd; do
  if [ "$v" = base ]; then lib=paper_2605_18334_b200/libssg_b200.so; else lib=paper_2605_18334_b200/libssg_b200_$v.so; fi
  echo "== $v c2" >> gpurun_out/r2x_ab.txt
  SSG_B200_LIB=$lib timeout 300 python tools/stage_times.py --reps 6 2>&1 | tail -2 | head -1 >> gpurun_out/r2x_ab.txt
  echo "== $v c4" >> gpurun_out/r2x_ab.txt
  SSG_B200_LIB=$lib timeout 300 python tools/stage_times.py --reps 6 --ball 2>&1 | tail -2 | head -1 >> gpurun_out/r2x_ab.txt
done
tail -3 gpurun_out/r2x_pytest.txt; cat gpurun_out/r2x_ab.txt
