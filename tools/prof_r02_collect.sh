#!/bin/bash
# Copy the products of tools/gpu_prof_r02.sh from gpurun_out/ into profiles/ (run here, after the call).
set -e
cd "$(dirname "$0")/.."
G=gpurun_out
cp $G/r02_bench_final.json profiles/r02_bench_line.json
cp $G/r02_kernel_traffic.json profiles/r02_kernel_traffic.json
for f in $G/r02_C*_lines.txt; do cp "$f" profiles/; done
python - <<'PY'
import glob, json, os
out = {"source": "ncu --set full --clock-control none --import-source on, one full-size wave (wave 2 of the "
                  "warm-up pass) of each timed stage kernel at the bench's 2^24-slot pool (tools/gpu_prof_r02.sh, "
                  "summarised by tools/ncu_summary.py); serialised cold-cache launches",
       "round": "r02", "kernels": {}}
for f in sorted(glob.glob("gpurun_out/r02_C*_summary.json")):
    key = os.path.basename(f)[4:-len("_summary.json")]
    rows = json.load(open(f))
    out["kernels"][key] = max(rows, key=lambda r: r["duration_us"])  # the full-size wave, not the flush
json.dump(out, open("profiles/r02_ncu_stage_kernels.json", "w"), indent=1)
PY
python tools/launch_summary.py $G/launches_C2.csv > profiles/r02_launch_shares_C2.txt
python tools/c3_waves.py $G/launches_C3.csv > profiles/r02_C3_waves.txt
echo collected
