"""Per-kernel share of GPU time from an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(d["Metric Unit"], 1e-3)
    name = d["Kernel Name"].split("(")[0]
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
print(f"{'kernel':58s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:16]:
    print(f"{k[:58]:58s} {cnt[k]:8d} {v:10.1f} {v / cnt[k]:9.2f} {100 * v / s:5.1f}%")
