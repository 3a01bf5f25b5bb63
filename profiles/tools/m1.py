"""Executed FP32 work of the force kernels (SURVEY 8(d) metric M1) from an ncu
CSV of the thread-level op counters (packed fp32x2 ops count two lanes):
flops = fadd + fmul + 2 ffma + 2 fadd2 + 2 fmul2 + 4 ffma2, divided by the
kernel duration and the FP32 peak (148 SMs x 128 lanes x 2 flop x clock)."""
import csv
import sys
from collections import defaultdict

W = {"fadd": 1, "fmul": 1, "ffma": 2, "fadd2": 2, "fmul2": 2, "ffma2": 4}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
names = {}
for r in rows[1:]:
    per[r[iid]][r[im]] = float(r[iv].replace(",", ""))
    names[r[iid]] = r[ik].split("(")[0]
peak_mhz = float(sys.argv[2]) if len(sys.argv) > 2 else 1965.0
for k, m in per.items():
    t = m.get("gpu__time_duration.sum", 0) * 1e-9
    fl = sum(w * m.get(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum", 0) for op, w in W.items())
    peak = 148 * 128 * 2 * peak_mhz * 1e6
    print(f"{names[k][:44]:44s} {t*1e6:9.1f} us  {fl/1e9:8.3f} GFLOP executed  {fl/t/1e12:6.2f} TFLOP/s  "
          f"M1 = {100*fl/t/peak:5.1f} % of {peak/1e12:.2f}")
