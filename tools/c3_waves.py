"""Per-wave device time of the stage kernels from an ncu launch list (C3 wave breakdown).

usage: python tools/c3_waves.py gpurun_out/launches_C3.csv > profiles/r02_C3_waves.txt
Takes the last pass that traced rays (a pass ends at k_fb_accumulate) and splits it at k_wave_begin.
"""
import csv
import sys

STAGES = [("generate", "k_generate"), ("trace_ext", "k_trace_ext_p"), ("shade_nee", "k_shade_nee"),
          ("shade", "k_shade<"), ("shadow", "k_trace_shadow_p")]
UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}

hdr, seq = None, []
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") == "gpu__time_duration.sum":
        seq.append((d["Kernel Name"].split("(")[0], float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1e-3)))

passes, cur = [], []
for name, us in seq:
    cur.append((name, us))
    if "k_fb_accumulate" in name:
        passes.append(cur)
        cur = []
traced = [p for p in passes if any("k_trace_ext_p" in n for n, _ in p)]
if not traced:
    sys.exit("no traced pass in the launch list")
last = traced[-1]
waves, w = [], None
for name, us in last:
    if "k_wave_begin" in name:
        w = dict.fromkeys([s for s, _ in STAGES], 0.0)
        waves.append(w)
    if w is None:
        continue
    for s, pat in STAGES:
        if pat in name:
            w[s] += us
print("# per-wave device time of the stage kernels in the last traced pass of "
      "`ncu --metrics gpu__time_duration.sum --clock-control none` (serialised, cold).")
print("# Wave 1 = primary rays (coherent), later waves secondaries.  A final generate-only wave flushes.")
print("wave " + "".join(f"{s:>11s}" for s, _ in STAGES) + "   (us)")
for i, w in enumerate(waves, 1):
    print(f"{i:4d} " + "".join(f"{w[s]:11.1f}" for s, _ in STAGES))
tot = {s: sum(w[s] for w in waves) for s, _ in STAGES}
allt = sum(tot.values())
print(f"trace_ext share of the stage-kernel time: {tot['trace_ext'] / allt:.3f}; "
      f"wave-1 (primary) share of trace_ext: {waves[0]['trace_ext'] / tot['trace_ext']:.3f}")
