"""A long decomposed run at full BASELINE size on one GPU: c4 (16.8 M molecules) on p loopback
ranks, rebalanced every 100 steps (BASELINE configs[4]), stepped for N steps.  Checks: no error,
molecule count and ids conserved, per-step global U / W / T against the one-domain GPU run of the
same system (same library, fp32 sums in another order: agreement to ~1e-5 while the two
trajectories stay together), boxes after each rebalance, owned-load imbalance.

  python profiles/tools/dd_longrun.py c4 8 250
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import scenarios as S  # noqa: E402
from paper_1408_4599_b200 import mardyn  # noqa: E402


def main():
    name, p, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    s = S.config(name)
    t = time.time()
    run = mardyn.DecomposedRun(s, p, transport="loopback", rebalance_interval=100)
    boxes0 = np.asarray(run.boxes).reshape(p, 6).tolist()
    run.step(n)
    hist = run.observable_history(n)
    wall = time.time() - t
    owned = run.owned_counts()
    ids = run.molecules()["id"]
    ref = mardyn.from_system(s)
    ref.step(n)
    rh = ref.get_observable_history(n)
    err = {}
    for key in ("U_pot", "virial", "T"):
        a = np.array([h[key] for h in hist]); b = np.array([h[key] for h in rh])
        e = np.abs(a - b) / np.abs(b).max()
        err[key] = {"max": float(e.max()), "at": int(e.argmax()), "first10": float(e[:10].max())}
    out = {"config": name, "p": p, "steps": n, "wall_s": round(wall, 1),
           "ids_conserved": bool(np.array_equal(np.sort(ids), np.arange(len(s["r"])))),
           "owned": owned, "owned_max_over_mean": float(max(owned) / np.mean(owned)),
           "boxes_initial": boxes0, "boxes_final": np.asarray(run.boxes).reshape(p, 6).tolist(),
           "vs_one_domain": err, "U_first_last": [hist[0]["U_pot"], hist[-1]["U_pot"]],
           "T_first_last": [hist[0]["T"], hist[-1]["T"]]}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
