#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_small.py
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 3 \
    python tools/sanitize_small.py > gpurun_out/${TAG:-r2b}_sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/${TAG:-r2b}_sanitize_$tool.txt
  tail -4 gpurun_out/${TAG:-r2b}_sanitize_$tool.txt
done
