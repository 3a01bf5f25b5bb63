"""The library's NCCL transport with several processes on ONE GPU, against the fp64 oracle.

A decomposed run over NCCL (mardyn_create_distributed: one rank per process, the library's
own communicator) normally needs one GPU per rank, and NCCL refuses two ranks of a
communicator on one device.  Here each rank is its own process on cuda:0 and the library
loads, through MARDYN_NCCL_LIB, the host-staged stand-in tests/nccl_shim.c (NCCL's entry
points and calling convention; every operation completed on the host; its own semantics
pinned by tests/test_nccl_shim_host.py).  So the code that only runs over NCCL executes with
the real kernels: the record counts of the first step all-gathered, the exact exchange by
grouped send / recv, the fixed per-peer segments with device-side counts of the
asynchronous steps, the cell loads all-reduced for the rebalance, the observables
all-gathered and summed in rank order, and the failure agreement before each collective of
the host-synchronous paths.  The oracle integrates the whole system (it knows nothing of
ranks).  Compared: every molecule's F(t0) and tau(t0) exactly once over the ranks, the
global U, W, T per step (1e-5, reading A25) and n_pairs, identical observables on every
rank, the ids after the run (migration conserves them) and the final positions (1e-4 sigma).
"""
import json
import os

import numpy as np
import pytest

from nccl_shim_util import build_shim
from parity_util import assert_forces_close, min_image

pytestmark = pytest.mark.gpu


def system(cfg):
    import scenarios as S
    return S.config3(12) if cfg == "c3m" else S.config(cfg)      # c3m: water, 6 912 molecules, 5^3 cells


def _rank_main(rank, world, port, shim, outdir, cfg, nsteps, rebalance, boxes, ipc):
    os.environ.update(MARDYN_NCCL_LIB=shim, MDSHIM_DIR=outdir, MDSHIM_LOG=outdir, MDSHIM_TIMEOUT_S="120",
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), MARDYN_IPC_PUTS="1" if ipc else "0")
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)    # launches ranks, carries the unique id
    torch.cuda.set_device(0)
    from paper_1408_4599_b200 import mardyn
    s = system(cfg)
    out = {"rank": rank}
    try:
        run = mardyn.DecomposedRun(s, world, transport="nccl", rank=rank, rebalance_interval=rebalance,
                                   boxes=None if boxes is None else np.asarray(boxes))
        F, tau, ids = run.forces()
        boxes0 = run.boxes.tolist()
        run.step(nsteps)
        hist = run.observable_history(nsteps)
        m = run.molecules()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), F=F, tau=tau, ids=ids, mid=m["id"], mr=m["r"])
        out.update(hist=hist, boxes0=boxes0, boxes1=run.boxes.tolist(), owned=run.owned_counts())
    except Exception as e:            # reported to the parent (every rank must fail alike)
        out["error"] = repr(e)
    with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
        json.dump(out, f)
    dist.destroy_process_group()


def run_ranks(tmp_path, world, cfg, nsteps, rebalance=0, boxes=None, ipc=True):
    import socket
    import torch.multiprocessing as tmp
    shim = build_shim(tmp_path)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    tmp.start_processes(_rank_main, args=(world, port, shim, str(tmp_path), cfg, nsteps, rebalance, boxes, ipc),
                        nprocs=world, join=True, start_method="spawn")
    res = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    for r in res:        # point-to-point messages this rank sent through the stand-in
        r["p2p_sends"] = sum(1 for l in open(tmp_path / f"shim_rank{r['rank']}.log") if l.startswith("send "))
    return res


def check_transport(res, world, nsteps, ipc, sync_steps=1):
    """IPC puts: point-to-point messages only in the synchronous steps (the exact exchange of
    the first step and of each rebalance); send / recv: four per peer in every other step."""
    for r in res:
        if ipc:
            assert r["p2p_sends"] <= 2 * (world - 1) * sync_steps, r["p2p_sends"]
        else:
            assert r["p2p_sends"] >= 2 * (world - 1) * (nsteps - sync_steps), r["p2p_sends"]


def shim_logs(tmp_path, n=12):
    out = []
    for f in sorted(os.listdir(tmp_path)):
        if f.startswith("shim_rank"):
            out.append(f + ":\n" + "".join(open(tmp_path / f).readlines()[-n:]))
    return "\n".join(out)


def check_against_oracle(oracle_mod, tmp_path, res, cfg, nsteps):
    for r in res:
        assert "error" not in r, (r, shim_logs(tmp_path))
    s = system(cfg)
    world = len(res)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    ids = np.concatenate([p["ids"] for p in parts])
    order = np.argsort(ids)
    assert np.array_equal(ids[order], np.arange(len(s["r"])))             # every molecule exactly once
    F = np.concatenate([p["F"] for p in parts])[order]
    tau = np.concatenate([p["tau"] for p in parts])[order]
    o = oracle_mod.System(s)
    u0 = o.quantize(s["r"])
    Fo, to, _ = o.forces(s["comp"], u0, s["q"], mode="full")
    assert_forces_close(F, Fo, "force(t0)")
    if any(c["charges"] or c["dipoles"] or c["quadrupoles"] for c in s["components"]):
        assert_forces_close(tau, to, "torque(t0)")
    hist = res[0]["hist"]
    for r in res[1:]:
        assert r["hist"] == hist                                          # global values on every rank
    uo, _, _, _, obs = o.run(s["dt"], s["comp"], u0, s["v"], s["q"], s["j"], nsteps, mode="full")
    assert [h["step"] for h in hist] == list(range(nsteps))
    for key, ok in (("U_pot", "U"), ("virial", "W"), ("T", "T")):
        ref = np.asarray(obs[ok], float)
        e = np.abs(np.array([h[key] for h in hist]) - ref) / np.abs(ref).max()
        assert e.max() <= 1e-5, (key, int(e.argmax()), e.max())
    npg = np.array([h["n_pairs"] for h in hist])
    assert npg[0] == obs["npairs"][0]
    assert (np.abs(npg - obs["npairs"]) <= np.maximum(2, 1e-5 * obs["npairs"])).all()
    mid = np.concatenate([p["mid"] for p in parts])
    mo = np.argsort(mid)
    assert np.array_equal(mid[mo], np.arange(len(s["r"])))                # ids conserved by migration
    mr = np.concatenate([p["mr"] for p in parts])[mo]
    assert np.abs(min_image(mr - uo * o.quantum, o.box)).max() <= 1e-4
    return hist


@pytest.fixture(scope="module")
def built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1408_4599_b200 import build
    build.build()
    return True


@pytest.mark.parametrize("ipc", [True, False])
def test_nccl_two_processes_lj(built, oracle_mod, tmp_path, ipc):
    """c1s (single-site LJ) on two processes: halo exchange and migration every step, the
    records stored by the fused force + leapfrog kernel straight into the peer's receive area
    (IPC puts), or moved by grouped send / recv (MARDYN_IPC_PUTS=0)."""
    res = run_ranks(tmp_path, 2, "c1s", 12, ipc=ipc)
    check_against_oracle(oracle_mod, tmp_path, res, "c1s", 12)
    check_transport(res, 2, 12, ipc)
    assert all(min(r["owned"]) > 0 for r in res)


@pytest.mark.parametrize("ipc", [True, False])
def test_nccl_three_processes_water_rebalance(built, oracle_mod, tmp_path, ipc):
    """Water (four sites, reaction field) on three processes from unequal boxes (a z slab and two halves of the rest),
    re-partitioned from the measured cell loads every 4 steps (all-reduce of the loads,
    redistribution through the exchange records)."""
    s = system("c3m")
    n = np.floor(np.asarray(s["box"]) / s["rc"]).astype(int)
    boxes = [[0, 0, 0, n[0], n[1], 2], [0, 0, 2, n[0], 2, n[2]], [0, 2, 2, n[0], n[1], n[2]]]
    res = run_ranks(tmp_path, 3, "c3m", 10, rebalance=4, boxes=boxes, ipc=ipc)
    check_against_oracle(oracle_mod, tmp_path, res, "c3m", 10)
    check_transport(res, 3, 10, ipc, sync_steps=3)           # the first step, after rebalances at 4 and 8
    assert res[0]["boxes1"] == res[1]["boxes1"] == res[2]["boxes1"]
    assert np.asarray(res[0]["boxes1"]).reshape(3, 6).tolist() != boxes          # re-partitioned


def test_nccl_four_processes_slab_rebalance(built, oracle_mod, tmp_path):
    """c4s (vapour-liquid slab) on four processes with rebalances every 3 steps."""
    res = run_ranks(tmp_path, 4, "c4s", 9, rebalance=3)
    check_against_oracle(oracle_mod, tmp_path, res, "c4s", 9)
    check_transport(res, 4, 9, True, sync_steps=3)


def test_bench_two_ranks_one_device(built, tmp_path):
    """bench.py's N > 1 path (torchrun, one rank per process, max over ranks, the e2e leg of a
    decomposed run) on one GPU: MARDYN_BENCH_ONE_DEVICE=1 puts every rank on cuda:0 with a
    gloo group and the library's transport on the stand-in.  The line reports n_gpus = 2 and
    the same observables as the one-GPU line of the same run length."""
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    shim = build_shim(tmp_path)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    args = ["--config", "c0", "--steps", "5", "--warmup", "3", "--e2e-steps", "2", "--no-cpu-baseline"]
    env = dict(os.environ, MARDYN_BENCH_ONE_DEVICE="1", MARDYN_NCCL_LIB=shim, MDSHIM_DIR=str(tmp_path))

    def line(cmd, env):
        out = subprocess.run(cmd, capture_output=True, text=True, cwd=root, env=env, timeout=900)
        assert out.returncode == 0, out.stderr[-3000:]
        ls = [l for l in out.stdout.splitlines() if l.startswith("{")]
        assert len(ls) == 1, out.stdout[-2000:]
        return json.loads(ls[0])

    d2 = line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2"] + args, env)
    d1 = line([sys.executable, "bench.py"] + args, dict(os.environ))
    assert d2["n_gpus"] == 2 and d2["value"] > 0 and d2["steps"] == 5
    assert "error" not in d2["e2e"] and d2["e2e"]["value"] > 0
    o1, o2 = d1["observables"], d2["observables"]
    assert o2["step"] == o1["step"] and o2["n_pairs"] == o1["n_pairs"]
    for k in ("U_pot", "virial", "T"):
        assert abs(o2[k] - o1[k]) <= 1e-5 * abs(o1[k]), (k, o1[k], o2[k])
