"""Per-rank device time of the decomposed step on ONE GPU (loopback ranks run one
after another on one stream, so each rank's own kernels are timed alone by CUDA
events around its begin / end halves; mardyn_last_step_timing total_ms).

  python profiles/tools/dd_ranks.py scale c4 1 2 4 8     # slowest rank vs T1 / p
  python profiles/tools/dd_ranks.py droplet 4 8          # static equal-volume vs k-d (Fig. 7 direction)

Prints one JSON line per measurement.  A number here is the kernel time of the
slowest rank of a p-GPU run; the exchange itself (NCCL over NVLink) is not in it.
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import scenarios as S  # noqa: E402
from paper_1408_4599_b200 import mardyn  # noqa: E402

import os  # noqa: E402

STEPS, WARM = int(os.environ.get("DD_STEPS", 20)), int(os.environ.get("DD_WARM", 4))
COST_MODEL = int(os.environ.get("DD_COST_MODEL", 0))      # 0: Eq. 6, 1: molecule counts (scale / one)


def t_single(s):
    import torch
    st = torch.cuda.Stream()
    ctx = mardyn.from_system(s, stream=st)
    ctx.step(WARM)
    ctx.get_observables()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms, fms = [], []
    for _ in range(STEPS):
        e0.record(st)
        ctx.step(1)
        e1.record(st)
        st.synchronize()
        ms.append(e0.elapsed_time(e1))
        fms.append(ctx.last_step_timing()["force_ms"])
    del ctx
    print(json.dumps({"single_force_ms": float(np.median(fms))}), flush=True)
    return float(np.median(ms))


def t_ranks(s, p, boxes=None, rebalance=0, cost_model=0):
    run = mardyn.DecomposedRun(s, p, transport="loopback", boxes=boxes, rebalance_interval=rebalance,
                               cost_model=cost_model)
    run.step(WARM)
    run.observables()
    per, fper = [], []
    for _ in range(STEPS):
        run.step(1)
        run.lead.stream.synchronize()
        tm = [c.last_step_timing() for c in run.ctxs]
        per.append([t["total_ms"] for t in tm])
        fper.append([t["force_ms"] for t in tm])
    per = np.array(per)
    med = np.median(per, axis=0)
    fmed = np.median(np.array(fper), axis=0)
    out = {"rank_ms": [round(float(x), 4) for x in med], "slowest_ms": float(med.max()),
           "force_ms": [round(float(x), 4) for x in fmed],
           "owned": run.owned_counts(), "boxes": np.asarray(run.boxes).reshape(p, 6).tolist()}
    del run
    return out


def equal_volume(s, p):
    n = np.floor(np.asarray(s["box"]) / s["rc"]).astype(int)
    cuts = [[0, n[0] // 2, n[0]], [0, n[1] // 2, n[1]] if p >= 4 else [0, n[1]],
            [0, n[2] // 2, n[2]] if p >= 8 else [0, n[2]]]
    return [[x0, y0, z0, x1, y1, z1] for z0, z1 in zip(cuts[2], cuts[2][1:])
            for y0, y1 in zip(cuts[1], cuts[1][1:]) for x0, x1 in zip(cuts[0], cuts[0][1:])]


def main():
    mode = sys.argv[1]
    if mode == "scale":
        name, ps = sys.argv[2], [int(x) for x in sys.argv[3:]]
        s = S.config(name)
        t1 = t_single(s)
        print(json.dumps({"config": name, "n": len(s["r"]), "p": 1, "T1_ms": t1}), flush=True)
        for p in ps:
            if p == 1:
                continue
            r = t_ranks(s, p, cost_model=COST_MODEL)
            r.update({"config": name, "p": p, "cost_model": COST_MODEL, "T1_over_p_ms": t1 / p,
                      "ratio": r["slowest_ms"] / (t1 / p)})
            print(json.dumps(r), flush=True)
    elif mode == "one":                     # one configuration, p ranks only (profiling)
        name, p = sys.argv[2], int(sys.argv[3])
        r = t_ranks(S.config(name), p)
        print(json.dumps(r), flush=True)
    elif mode == "static":                  # Fig. 7 direction on the slab: static z-slabs / octants vs k-d
        name = sys.argv[2]
        s = S.config(name)
        n = np.floor(np.asarray(s["box"]) / s["rc"]).astype(int)
        for p in [int(x) for x in sys.argv[3:]]:
            zc = [round(k * n[2] / p) for k in range(p + 1)]
            slabs = [[0, 0, zc[k], n[0], n[1], zc[k + 1]] for k in range(p)]
            out = {"config": name, "p": p}
            for lab, bx in (("zslab", slabs), ("octant", equal_volume(s, p)), ("kd", None)):
                r = t_ranks(s, p, boxes=bx)
                out[lab + "_slowest_ms"] = r["slowest_ms"]
                out[lab + "_owned_max_over_mean"] = float(max(r["owned"]) / np.mean(r["owned"]))
                out[lab + "_rank_ms"] = r["rank_ms"]
            out["zslab_over_kd"] = out["zslab_slowest_ms"] / out["kd_slowest_ms"]
            print(json.dumps(out), flush=True)
    elif mode == "droplet":
        t = time.time()
        s = S.droplet(L=320.0, R=85.0)          # ~2.5 M molecules; R / L < 0.3 keeps the sphere off the seam
        print(json.dumps({"droplet_n": len(s["r"]), "gen_s": time.time() - t}), flush=True)
        t1 = t_single(s)
        counts = mardyn.grid_counts(s["box"], s["rc"], s["r"]).astype(np.float64)
        for p in [int(x) for x in sys.argv[2:]]:
            st = t_ranks(s, p, boxes=equal_volume(s, p))
            kd = t_ranks(s, p)
            # the same tree on plain molecule counts (cost model 1) and on Eq. 6 + alpha N_i
            kdn = t_ranks(s, p, cost_model=1)
            eq6 = mardyn.cell_cost(counts.astype(np.int32))
            alt = {}
            for alpha in (100.0, 300.0):
                bA, _ = mardyn.kd_decompose(eq6 + alpha * counts, p)
                alt[alpha] = t_ranks(s, p, boxes=bA.reshape(p, 6))["slowest_ms"]
            print(json.dumps({"p": p, "kd_counts_slowest_ms": kdn["slowest_ms"], "kd_counts_rank_ms": kdn["rank_ms"],
                              "kd_eq6_alpha_slowest_ms": alt}), flush=True)
            print(json.dumps({"config": "droplet", "n": len(s["r"]), "p": p, "T1_ms": t1,
                              "static_slowest_ms": st["slowest_ms"], "kd_slowest_ms": kd["slowest_ms"],
                              "static_over_kd": st["slowest_ms"] / kd["slowest_ms"],
                              "static_owned": st["owned"], "kd_owned": kd["owned"],
                              "static_rank_ms": st["rank_ms"], "kd_rank_ms": kd["rank_ms"]}), flush=True)


if __name__ == "__main__":
    main()
