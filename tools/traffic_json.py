"""profiles/trace_ext_traffic.json from gpurun_out/traffic_<cfg>.csv (tools/gpu_evidence.sh).

Mean DRAM bytes (read + write) and duration per launch of the timed instantiation
k_trace_ext[_p]<false, ...> (the counting instantiation <true> runs only in bench.py's untimed pass).
"""
import collections
import re
import csv
import glob
import json
import os
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
        "msecond": 1e3, "ms": 1e3}
out = {}
for path in sorted(glob.glob("gpurun_out/traffic_C*.csv")):
    cfg = os.path.basename(path)[8:-4]
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(dict)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if not re.search(r"k_trace_ext(_p)?<(0|false)\b", d["Kernel Name"]):
            continue
        per[d["ID"]][d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
    recs = [v for v in per.values() if len(v) == 3]
    if not recs:
        continue
    n = len(recs)
    rd = sum(v["dram__bytes_read.sum"] for v in recs) / n
    wr = sum(v["dram__bytes_write.sum"] for v in recs) / n
    us = sum(v["gpu__time_duration.sum"] for v in recs) / n
    out[cfg] = {"launches": n, "dram_read_bytes_per_launch": rd, "dram_write_bytes_per_launch": wr,
                "dram_bytes_per_launch": rd + wr, "duration_us_per_launch": us,
                "dram_gbs": (rd + wr) / us / 1e3}
meta = {"kernel": "k_trace_ext_p<false, placement> (k_trace_ext<false, placement> with LW_TRACE_PERSIST=0)", "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
        "dram__bytes_write.sum --clock-control none (tools/gpu_evidence.sh); serialised, cold-cache launches",
        "round": sys.argv[1] if len(sys.argv) > 1 else "r01", "configs": out}
json.dump(meta, open("profiles/trace_ext_traffic.json", "w"), indent=1)
print(json.dumps(meta, indent=1))
