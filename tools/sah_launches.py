"""Per-kernel device time of the first SAH build in an ncu launch list (tools: ncu --metrics
gpu__time_duration.sum --csv ... python tools/e2e_breakdown.py C3)."""
import collections
import csv
import sys

hdr, seq = None, []
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") == "gpu__time_duration.sum":
        seq.append((d["Kernel Name"].split("(")[0].split("::")[-1], float(d["Metric Value"].replace(",", "")) / 1e3,
                    d.get("Grid Size", "")))
i0 = next(i for i, x in enumerate(seq) if "k_sah_prep" in x[0])
i1 = next(i for i, x in enumerate(seq) if "k_collapse_level" in x[0] and i > i0)
tot, cnt = collections.defaultdict(float), collections.Counter()
for n, t, g in seq[i0:i1]:
    tot[n[:40]] += t
    cnt[n[:40]] += 1
print("SAH build kernels: %.1f us in %d launches" % (sum(tot.values()), sum(cnt.values())))
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print("%9.1f %5d %s" % (v, cnt[k], k))
if "-v" in sys.argv:
    for n, t, g in seq[i0:i1]:
        if "decide" in n or "bin_large" in n:
            print("%-20s %8.1f %s" % (n[:20], t, g))
