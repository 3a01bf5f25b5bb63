"""Longer decomposed runs over the library's NCCL path (IPC puts) with ranks as processes on
one GPU (the NCCL-API stand-in, tests/nccl_shim.c), against the oracle: c1s on 3 processes
for 100 steps, the c4s slab on 4 processes for 60 steps with rebalances every 10."""
import os
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle  # noqa: E402  (test infrastructure: the checker)
import test_gpu_nccl_shim as T  # noqa: E402


def main():
    oracle.build()
    for cfg, world, nsteps, reb in (("c1s", 3, 100, 0), ("c4s", 4, 60, 10)):
        with tempfile.TemporaryDirectory() as d:
            tmp = Path(d)
            res = T.run_ranks(tmp, world, cfg, nsteps, rebalance=reb, ipc=True)
            hist = T.check_against_oracle(oracle, tmp, res, cfg, nsteps)
            print(f"{cfg}: {world} processes, {nsteps} steps, rebalance every {reb or '-'}: per-step U/W/T "
                  f"within 1e-5 of the oracle, ids conserved, positions within 1e-4; p2p sends per rank "
                  f"{[r['p2p_sends'] for r in res]}; U(last) = {hist[-1]['U_pot']:.6f}", flush=True)


if __name__ == "__main__":
    main()
