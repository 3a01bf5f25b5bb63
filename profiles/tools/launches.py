import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; data = rows[1:]
ik = h.index("Kernel Name"); iv = h.index("Metric Value")
agg = collections.OrderedDict()
for r in data:
    k = r[ik].split("(")[0][:60]
    t = float(r[iv].replace(",", ""))
    c, s = agg.get(k, (0, 0.0))
    agg[k] = (c + 1, s + t)
tot = sum(s for c, s in agg.values())
for k, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:60s} {c:4d} {s/1e3:9.1f} us  avg {s/c/1e3:8.1f} us  {100*s/tot:5.1f}%")
