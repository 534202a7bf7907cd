#!/bin/bash
# Measure the FP64 FMA peak with the SM clock sampled during the run (nvidia-smi, 50 ms), and the
# latency/occupancy sweep.  Writes profiles/fp64_peak.json and gpurun_out/fp64_sweep.jsonl.
set -e
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw --format=csv,noheader,nounits -lms 50 > gpurun_out/fp64_clocks.csv &
SMI=$!
sleep 0.3
for i in 1 2 3; do tools/fp64_peak > gpurun_out/fp64_peak_$i.json; done
kill $SMI || true
tools/fp64_peak sweep > gpurun_out/fp64_sweep.jsonl
python - <<'PY'
import json, statistics
runs = [json.load(open(f"gpurun_out/fp64_peak_{i}.json")) for i in (1, 2, 3)]
clk = [l.split(",") for l in open("gpurun_out/fp64_clocks.csv") if l.strip()]
sm = [float(c[0]) for c in clk]
busy = [float(c[0]) for c in clk if float(c[3]) > 300] or sm
out = {"fp64_fma_tflops": max(r["fp64_fma_tflops"] for r in runs), "runs": [r["fp64_fma_tflops"] for r in runs],
       "sms": runs[0]["sms"], "how": "tools/fp64_peak: 148 SMs x 8 blocks x 256 threads, 8 independent DFMA chains "
       "per thread, best of 5 launches, best of 3 runs",
       "clocks": {"sm_mhz_median_under_load": statistics.median(busy), "sm_max_mhz": float(clk[0][1]),
                  "samples": len(clk), "reasons": sorted({c[2].strip() for c in clk})}}
json.dump(out, open("gpurun_out/fp64_peak.json", "w"), indent=1)  # copy to profiles/ by hand
print(json.dumps(out))
PY
cat gpurun_out/fp64_sweep.jsonl
