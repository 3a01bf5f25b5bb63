"""Achieved DRAM bandwidth of the bandwidth kernels (sort, scan, scatter, canonical gather,
integrator, finalize) from an ncu CSV of gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum, lts__t_bytes.sum (one row per launch and metric; lines not starting
with '"' -- the program's own output -- are skipped).  Peak: MEASURED_PEAKS-style copy
bandwidth given as argv[2] (GB/s), default 6550."""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')) if len(r) > 10]
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6550.0
h = rows[0]
ik, im, iv, iu, iid = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
         "ns": 1, "us": 1e3, "ms": 1e6}
per, name = collections.defaultdict(dict), {}
for r in rows[1:]:
    per[r[iid]][r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
    name[r[iid]] = r[ik].split("(")[0]
agg = collections.defaultdict(list)
for k, m in per.items():
    agg[name[k]].append(m)
for n, ms in agg.items():
    t = sum(m["gpu__time_duration.sum"] for m in ms) / len(ms)
    b = sum(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in ms) / len(ms)
    l2 = sum(m.get("lts__t_bytes.sum", 0) for m in ms) / len(ms)
    print(f"{n[:34]:34s} x{len(ms)} {t / 1e3:8.1f} us  DRAM {b / 1e6:7.1f} MB  {b / t:7.1f} GB/s "
          f"({100 * b / t / peak:5.1f} % of {peak:.0f})  L2 {l2 / 1e6:7.1f} MB")
