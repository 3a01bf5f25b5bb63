"""Where the end-to-end step (bench.py `e2e`) spends its time: set_molecules from pinned
host buffers, step(1), get_observables, get_molecules into pinned host buffers, each
timed by the wall clock around the call (each call ends with a stream synchronize),
plus the plain pinned-memory copy rates of the same byte counts (the PCIe floor).

  python profiles/tools/e2e_parts.py c1 [reps]
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import scenarios as S  # noqa: E402
from paper_1408_4599_b200 import mardyn  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    s = S.config(name)
    N = len(s["r"])
    ctx = mardyn.from_system(s)
    ctx.step(3)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    h_r, h_v, h_c, h_id = pin(s["r"]), pin(s["v"]), pin(s["comp"]), pin(s["id"])
    rigid = ctx.get_grid()["kernel"] != 0
    h_q = pin(s["q"]) if rigid else None
    h_j = pin(s["j"]) if rigid else None
    out = {"r": torch.empty((N, 3), dtype=torch.float64).pin_memory(),
           "v": torch.empty((N, 3), dtype=torch.float64).pin_memory()}
    if rigid:
        out["q"] = torch.empty((N, 4), dtype=torch.float64).pin_memory()
        out["j"] = torch.empty((N, 3), dtype=torch.float64).pin_memory()
    parts = {"set_molecules": [], "step": [], "get_observables": [], "get_molecules": [], "total": []}
    for k in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.set_molecules(h_r, h_v, comp=h_c, q=h_q, j=h_j, id=h_id, half_step=1)
        t1 = time.perf_counter()
        ctx.step(1)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ctx.get_observables()
        t3 = time.perf_counter()
        ctx.get_molecules(out)
        t4 = time.perf_counter()
        if k:
            for key, a, b in (("set_molecules", t0, t1), ("step", t1, t2), ("get_observables", t2, t3),
                              ("get_molecules", t3, t4), ("total", t0, t4)):
                parts[key].append((b - a) * 1e3)
    res = {k: round(float(np.median(v)), 4) for k, v in parts.items()}
    # the PCIe floor: the same bytes as plain pinned <-> device copies
    h2d_b = N * (3 * 8 + 3 * 8 + 4 + 8 + (7 * 8 if rigid else 0))
    d2h_b = N * (3 * 8 + 3 * 8 + (7 * 8 if rigid else 0))
    hb = torch.empty(h2d_b, dtype=torch.uint8).pin_memory()
    db = torch.empty(h2d_b, dtype=torch.uint8, device="cuda")
    hob = torch.empty(d2h_b, dtype=torch.uint8).pin_memory()
    ms_h, ms_d = [], []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        db.copy_(hb, non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        hob.copy_(db[:d2h_b], non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ms_h.append((t1 - t0) * 1e3)
        ms_d.append((t2 - t1) * 1e3)
    res.update({"config": name, "n": N, "h2d_bytes": h2d_b, "d2h_bytes": d2h_b,
                "h2d_copy_ms": round(float(np.median(ms_h)), 4), "d2h_copy_ms": round(float(np.median(ms_d)), 4),
                "h2d_GBps": round(h2d_b / np.median(ms_h) / 1e6, 1), "d2h_GBps": round(d2h_b / np.median(ms_d) / 1e6, 1)})
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
