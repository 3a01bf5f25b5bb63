import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
ia = h.index("Address"); isrc = h.index("Source"); iex = h.index("Instructions Executed"); ist = h.index("Warp Stall Sampling (All Samples)")
base = int(data[0][ia], 16)
tot = sum(int(r[iex]) for r in data); stot = sum(int(r[ist]) for r in data)
print("total inst", tot, "samples", stot)
# loops: backward branches
lst = []
for r in data:
    s = r[isrc].strip()
    if "BRA" in s:
        try:
            tgt = int(s.split("BRA")[1].strip().split()[0].rstrip(";"), 16) - base
        except Exception:
            continue
        me = int(r[ia], 16) - base
        if tgt < me:
            seg = [x for x in data if tgt <= int(x[ia], 16) - base <= me]
            lst.append((me, tgt, int(r[iex]), sum(int(x[iex]) for x in seg), sum(int(x[ist]) for x in seg), len(seg)))
for me, tgt, trips, ins, st, n in lst:
    print(f"loop {hex(tgt)}-{hex(me)} len {n:4d} trips {trips:9d} inst {ins:10d} ({100*ins/tot:5.1f}%) stall {100*st/stot:5.1f}%")
if len(sys.argv) > 2:
    a, b = int(sys.argv[2], 16), int(sys.argv[3], 16)
    for r in data:
        o = int(r[ia], 16) - base
        if a <= o <= b:
            print(hex(o), r[isrc][:70].ljust(70), r[iex], r[ist])
