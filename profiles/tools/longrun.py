"""Diagnostic: full-length GPU trajectories against the fp64 oracle, with the
oracle's own sensitivity (one-quantum perturbed oracle runs) alongside."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
import oracle, scenarios as S
from paper_1408_4599_b200 import mardyn as md

out = {}
for name, n in [a.split(":") for a in sys.argv[1:]]:
    n = int(n)
    s = S.config(name)
    t = time.time()
    ctx = md.from_system(s)
    ctx.step(n)
    h = ctx.get_observable_history(n)
    ug, cg, ng = ctx.get_raw()
    tg = time.time() - t
    o = oracle.System(s)
    u0 = o.quantize(s["r"])
    t = time.time()
    uo, vo, qo, jo, a = o.run(s["dt"], s["comp"], u0, s["v"], s["q"], s["j"], n, mode="full")
    to = time.time() - t
    up = u0.copy(); up[::7, 0] += 1
    _, _, _, _, b = o.run(s["dt"], s["comp"], up, s["v"], s["q"], s["j"], n, mode="full")
    co, no = o.cells(ug)
    res = {"n": len(u0), "gpu_s": tg, "oracle_s": to, "cells_exact": bool(np.array_equal(cg, co) and np.array_equal(ng, no)),
           "same_u": int((ug == uo).all(1).sum())}
    for k, gk in (("U", "U_pot"), ("W", "virial"), ("T", "T")):
        g = np.array([x[gk] for x in h])
        rg = np.abs(g - a[k]) / np.abs(a[k])
        rp = np.abs(b[k] - a[k]) / np.abs(a[k])
        res[k] = {"gpu_max": float(rg.max()), "gpu_argmax": int(rg.argmax()), "pert_max": float(rp.max()),
                  "gpu_at": [float(rg[i]) for i in (9, 19, 49, n - 1) if i < n],
                  "pert_at": [float(rp[i]) for i in (9, 19, 49, n - 1) if i < n]}
    res["npairs_equal_steps"] = int(sum(int(h[k]["n_pairs"] == a["npairs"][k]) for k in range(n)))
    out[name] = res
    print(name, json.dumps(res), flush=True)
