"""profiles/r02_kernel_traffic.json from gpurun_out/ktraffic_<cfg>.csv (tools/gpu_kernel_traffic.sh).

Per config and stage kernel (timed instantiation: COUNT template argument false), mean ncu DRAM
bytes (read + write) and duration per launch, and the launch-weighted DRAM throughput.
"""
import collections
import csv
import glob
import json
import os
import re

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
        "msecond": 1e3, "ms": 1e3}
# timed instantiations only (the <true>/<1> COUNT variants run in bench.py's untimed pass)
PATTERNS = {
    "k_generate": r"k_generate<(0|false)[,>]",
    "k_trace_ext_p": r"k_trace_ext(_p)?<(0|false), ",
    "k_shade_nee": r"k_shade_nee<",
    "k_shade": r"k_shade<",
    "k_trace_shadow_p": r"k_trace_shadow(_p)?<(0|false), ",
}
out = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 "--clock-control none (tools/gpu_kernel_traffic.sh), bench.py default pool (2^24 slots); "
                 "serialised cold-cache launches", "round": "r02", "configs": {}}
for path in sorted(glob.glob("gpurun_out/ktraffic_C*.csv")):
    cfg = os.path.basename(path)[9:-4]
    hdr = None
    per = collections.defaultdict(dict)
    names = {}
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        per[d["ID"]][d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        names[d["ID"]] = d["Kernel Name"]
    res = {}
    for key, pat in PATTERNS.items():
        recs = [v for i, v in per.items() if re.search(pat, names[i]) and len(v) == 3]
        if not recs:
            continue
        n = len(recs)
        rd = sum(v["dram__bytes_read.sum"] for v in recs) / n
        wr = sum(v["dram__bytes_write.sum"] for v in recs) / n
        us = sum(v["gpu__time_duration.sum"] for v in recs) / n
        res[key] = {"launches": n, "dram_read_bytes_per_launch": rd, "dram_write_bytes_per_launch": wr,
                    "dram_bytes_per_launch": rd + wr, "duration_us_per_launch": us,
                    "dram_gbs": (rd + wr) / (us * 1e3)}
    if res:
        tot = sum(v["duration_us_per_launch"] * v["launches"] for v in res.values())
        for v in res.values():
            v["share_of_stage_kernel_time"] = v["duration_us_per_launch"] * v["launches"] / tot
        out["configs"][cfg] = res
print(json.dumps(out, indent=1))
