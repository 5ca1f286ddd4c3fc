"""profiles/r01_ncu_stage_kernels.json from the ncu reports of tools/gpu_prof_final.sh."""
import glob
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import load  # noqa: E402

rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = {}
for path in sorted(glob.glob(f"gpurun_out/{rnd}_C*_*.ncu-rep")):
    name = os.path.basename(path)[len(rnd) + 1:-8]
    recs = load(path)
    if recs:
        out[name] = recs[0]
meta = {"round": rnd,
        "command": "tools/gpu_prof_final.sh: ncu --set full --clock-control none --import-source on, one steady-state "
                   "launch per kernel (python bench.py --steps 1 --warmup 1 --config Cn; default 2^23-slot pool); "
                   "timed instantiations only",
        "note": "durations are serialised single-launch ncu times; Cornell-box (C1/C2) trace kernels read the BVH "
                "from shared memory, so their DRAM bytes are the SoA ray state",
        "kernels": out}
json.dump(meta, open(f"profiles/{rnd}_ncu_stage_kernels.json", "w"), indent=1)
for k, v in out.items():
    print(k, v["duration_us"], "issue", v.get("issue_active_pct"), "l1tex", v.get("l1tex_throughput_pct"))
