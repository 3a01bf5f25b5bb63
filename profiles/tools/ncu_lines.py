import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = None; per = collections.Counter(); st = collections.Counter(); src = {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    # cuda line rows have Address empty? each row: line, source, address, sass, stall...
    iex = hdr.index("Instructions Executed"); ist = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        per[(fname, ln)] += int(r[iex] or 0); st[(fname, ln)] += int(r[ist] or 0)
    except ValueError:
        pass
    src[(fname, ln)] = r[1]
tot = sum(per.values()); stot = sum(st.values())
print("total", tot, stot)
for k, v in sorted(per.items(), key=lambda kv: -st[kv[0]])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{k[0]}:{k[1]:4d} inst {100*v/tot:5.1f}% stall {100*st[k]/stot:5.1f}%  {src[k].strip()[:80]}")
