"""L1TEX request / wavefront / sector breakdown (global vs local vs shared) from a raw ncu csv.

    python tools/l1tex_breakdown.py gpurun_out/X_raw.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, v = rows[0], rows[2]
m = dict(zip(h, v))


def g(k):
    try:
        return float(m.get(k, "0").replace(",", ""))
    except ValueError:
        return 0.0


print("kernel", m.get("Kernel Name", "?")[:80], " duration_ms", g("gpu__time_duration.sum") / (1e6 if "ns" in rows[1][h.index("gpu__time_duration.sum")] else 1e3))
for space, ops in (("global", ("ld", "st")), ("local", ("ld", "st"))):
    for op in ops:
        k = f"pipe_lsu_mem_{space}_op_{op}"
        print(f"{space:6s} {op}: requests {g('l1tex__t_requests_' + k + '.sum'):.3e} wavefronts "
              f"{g('l1tex__t_output_wavefronts_' + k + '.sum'):.3e} sectors {g('l1tex__t_sectors_' + k + '.sum'):.3e} "
              f"hit {g('l1tex__t_sector_' + k + '_hit_rate.pct'):.1f}%")
print(f"shared wavefronts {g('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum'):.3e}")
print(f"l1tex throughput {g('l1tex__throughput.avg.pct_of_peak_sustained_active'):.1f}%  dram read "
      f"{g('dram__bytes_read.sum'):.3e} write {g('dram__bytes_write.sum'):.3e}")
