"""Summarise an ncu --set full report: one JSON line of key metrics per kernel launch.

    python tools/ncu_summary.py gpurun_out/prof_trace.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "regs": "launch__registers_per_thread",
    "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_bytes": "lts__t_bytes.sum",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "threads_per_warp_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "local_ld_sectors": "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum",
    "l1tex_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "warp_instructions": "smsp__inst_executed.sum",
}
_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
_TIME = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    unit = dict(zip(hdr, units))
    res = []
    for r in data:
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")[:70]}
        for k, m in METRICS.items():
            v = d.get(m)
            if v in (None, "", "n/a"):
                continue
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            u = unit.get(m, "")
            x *= _TIME.get(u, 1.0) if k == "duration_us" else _BYTES.get(u, 1.0)
            rec[k] = round(x, 4)
        stalls = []
        for h in hdr:
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(d[h].replace(",", "")), h[34:-23]))
                except ValueError:
                    pass
        rec["top_stalls_per_issue"] = {n: round(v, 3) for v, n in sorted(stalls, reverse=True)[:5]}
        res.append(rec)
    return res


if __name__ == "__main__":
    recs = load(sys.argv[1])
    for r in recs:
        print(json.dumps(r))
    if "--json" in sys.argv:
        json.dump(recs, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
