#!/bin/bash
# Measure FP32 FFMA / MUFU ex2 / MUFU rcp lane throughput on the GPU box and
# write profiles/measured_issue_peaks.json (SM clock sampled during the run).
set -e
cd "$(dirname "$0")/../.."
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ssg_peaks tools/micro/peaks.cu
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv,noheader,nounits \
    -lms 100 > /tmp/ssg_peaks_clk.txt &
SMI=$!
sleep 0.5
/tmp/ssg_peaks > /tmp/ssg_peaks.json
kill $SMI
python - <<'PY'
import json, statistics
r = json.load(open("/tmp/ssg_peaks.json"))
rows = [l.split(",") for l in open("/tmp/ssg_peaks_clk.txt") if l.strip()]
sm = [float(x[0]) for x in rows]
r["sm_mhz_samples"] = len(sm)
r["sm_mhz_max_seen"] = max(sm) if sm else None
r["sm_mhz_median"] = statistics.median(sm) if sm else None
r["sm_max_mhz"] = float(rows[0][1]) if rows else None
f = r["sm_mhz_max_seen"] or r["clock_rate_mhz_attr"]
for k in ("ffma", "ex2", "rcp"):
    r[k + "_per_sm_clk"] = r[k + "_lane_per_s"] / r["sms"] / (f * 1e6)
r["how"] = "tools/micro/peaks.cu: 8 independent chains/thread, 8x256 threads per SM, best of 5 launches (CUDA events)"
json.dump(r, open("profiles/measured_issue_peaks.json", "w"), indent=1)
print(json.dumps(r))
PY
