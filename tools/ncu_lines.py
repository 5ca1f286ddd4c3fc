"""Per-source-line hot spots of one kernel from an ncu report (needs -lineinfo + --import-source).

    python tools/ncu_lines.py report.ncu-rep <kernel-regex> [top]
Prints (share of stall samples, share of warp instructions, file:line, source) for the top lines.
"""
import csv
import io
import os
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
path, hdr, recs = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue  # sass row under a source line
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = float(d.get("Warp Stall Sampling (All Samples)", "0").replace(",", "") or 0)
        i = float(d.get("Instructions Executed", "0").replace(",", "") or 0)
    except ValueError:
        continue
    recs.append((s, i, f"{path}:{r[0]}", r[1].strip()))
S = sum(x[0] for x in recs) or 1
I = sum(x[1] for x in recs) or 1
print(f"samples {S:.0f} warp-instructions {I:.3e}")
for s, i, loc, src in sorted(recs, reverse=True)[:top]:
    print(f"{s / S:6.1%} {i / I:6.1%} {loc:<26} {src[:90]}")
