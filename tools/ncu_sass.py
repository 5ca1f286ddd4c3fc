"""Stall summary of one kernel from an ncu report's SASS source page.

    python tools/ncu_sass.py report.ncu-rep <kernel-regex> [top]
Prints the stall-reason totals and the instructions with the most warp-stall samples.
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


tot = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print(f"instructions {len(data)}  samples {tot:.0f}")
agg = sorted(((sum(f(d[s]) for d in data), s) for s in stalls), reverse=True)
print("  ".join(f"{s[6:]} {v / tot:.1%}" for v, s in agg if v > 0.005 * tot))
inst = sum(f(d["Instructions Executed"]) for d in data)
thr = sum(f(d["Thread Instructions Executed"]) for d in data)
print(f"warp instructions {inst:.3e}  avg threads/inst {thr / max(inst, 1):.2f}")
data.sort(key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))
for d in data[:top]:
    s = f(d["Warp Stall Sampling (All Samples)"])
    main = max(stalls, key=lambda k: f(d[k]))
    print(f"{d['Address']:>6} {s / tot:6.1%} thr {f(d['Avg. Threads Executed']):5.1f} {main[6:]:<14} {d['Source'][:80]}")
