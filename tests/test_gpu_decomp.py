"""Spatial decomposition (§4) against the fp64 oracle.

p ranks of one decomposition run on one GPU as a loopback group
(mardyn_create_loopback: k-d boxes, one halo cell layer, migration, records
stored straight into the receiving rank's buffers -- the library's own
exchange, rebalance and global observables).  The oracle knows
nothing of the decomposition: it integrates the whole system.  Compared per
step: the GLOBAL U, W, T (reading A25 measure, 1e-5) and n_pairs, the forces
of t_0 per molecule (A15), the molecule count and ids (migration conserves
them), and the final positions (1e-4 sigma).  The rebalance cases re-partition
from the measured per-cell loads during the run.
"""
import numpy as np
import pytest

import scenarios as S
from parity_util import assert_forces_close, min_image

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def md():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1408_4599_b200 import build, mardyn
    build.build()
    return mardyn


def scaled_err(a, b):
    b = np.asarray(b, float)
    return np.abs(np.asarray(a, float) - b) / np.abs(b).max()


def compare_run(md, oracle_mod, s, run, nsteps, tol=1e-5, eta=None):
    """Step the decomposed run and the oracle independently from the same state."""
    F, tau, ids = run.forces()                         # F(t0), tau(t0): every molecule exactly once
    assert np.array_equal(ids, np.arange(len(s["r"])))
    o = oracle_mod.System(s, eta=eta)
    u0 = o.quantize(s["r"])
    Fo, to, _ = o.forces(s["comp"], u0, s["q"], mode="full")
    assert_forces_close(F, Fo, "force(t0)")
    if any(c["charges"] or c["dipoles"] or c["quadrupoles"] for c in s["components"]):
        assert_forces_close(tau, to, "torque(t0)")
    run.step(nsteps)
    hist = run.observable_history(nsteps)
    uo, vo, qo, jo, obs = o.run(s["dt"], s["comp"], u0, s["v"], s["q"], s["j"], nsteps, mode="full")
    assert [h["step"] for h in hist] == list(range(nsteps))
    for key, ok in (("U_pot", "U"), ("virial", "W"), ("T", "T")):
        e = scaled_err([h[key] for h in hist], obs[ok])
        assert e.max() <= tol, (key, int(e.argmax()), e.max())
    npg = np.array([h["n_pairs"] for h in hist])
    assert npg[0] == obs["npairs"][0]
    assert (np.abs(npg - obs["npairs"]) <= np.maximum(2, 1e-5 * obs["npairs"])).all()
    m = run.molecules()
    assert np.array_equal(m["id"], np.arange(len(s["r"])))      # count and ids conserved
    assert np.abs(min_image(m["r"] - uo * o.quantum, o.box)).max() <= 1e-4
    return hist, obs


@pytest.mark.parametrize("name,p,nsteps", [("c1s", 2, 20), ("c1s", 3, 20), ("c4s", 4, 30), ("c4s", 8, 30),
                                           ("c2s", 4, 12), ("c3m", 2, 12)])
def test_decomposed_vs_oracle(md, oracle_mod, name, p, nsteps):
    # c3m: the water model on FCC 12^3 (6912 molecules, 5 cells per axis: c3s has 3, too
    # few for two boxes of >= 2 cells)
    s = S.config3(12) if name == "c3m" else S.config(name)
    run = md.DecomposedRun(s, p, transport="loopback")
    compare_run(md, oracle_mod, s, run, nsteps)


def equal_volume_boxes(s, p):
    """Static equal-volume boxes (halves along x, then y, then z)."""
    n = np.floor(np.asarray(s["box"]) / s["rc"]).astype(int)
    cuts = [[0, n[0] // 2, n[0]], [0, n[1] // 2, n[1]] if p >= 4 else [0, n[1]],
            [0, n[2] // 2, n[2]] if p >= 8 else [0, n[2]]]
    return [[[x0, y0, z0], [x1, y1, z1]] for z0, z1 in zip(cuts[2], cuts[2][1:])
            for y0, y1 in zip(cuts[1], cuts[1][1:]) for x0, x1 in zip(cuts[0], cuts[0][1:])]


@pytest.mark.parametrize("cost_model", [0, 1])
def test_rebalance_droplet_vs_oracle(md, oracle_mod, cost_model):
    """Off-centre droplet on 4 ranks starting from equal-volume
    boxes, re-partitioned every 5 steps from the measured cell loads (Eq. 6 or the
    molecule count): the owned-load imbalance drops, the boxes change, and every step
    still matches the oracle."""
    s = S.config("droplet")
    static = equal_volume_boxes(s, 4)
    run = md.DecomposedRun(s, 4, transport="loopback", boxes=static, rebalance_interval=5, cost_model=cost_model)
    before = run.owned_counts()
    compare_run(md, oracle_mod, s, run, 12)
    after = run.owned_counts()
    assert sum(after) == len(s["r"])
    assert max(after) / np.mean(after) < max(before) / np.mean(before) - 0.2
    assert not np.array_equal(np.asarray(run.boxes), np.asarray(static))


def test_decomposed_fullsize_c1_vs_oracle(md, oracle_mod):
    """The N > 1 bench workload at full size: c1 (1 048 576 molecules, BASELINE configs[1]) on
    8 ranks -- k-d boxes, halo exchange and migration every step -- for its full 100-step run
    against the oracle's one-domain run (F(t0) per molecule, per-step global U, W, T and
    n_pairs, ids, final positions)."""
    s = S.config("c1")
    run = md.DecomposedRun(s, 8, transport="loopback")
    compare_run(md, oracle_mod, s, run, 100)


def test_decomposed_fullsize_c4_vs_oracle(md, oracle_mod):
    """The slab at full size: c4 (16.8 M molecules, liquid and vapour, BASELINE configs[4]) on
    8 ranks for 5 steps against the oracle's one-domain run."""
    s = S.config("c4")
    run = md.DecomposedRun(s, 8, transport="loopback")
    compare_run(md, oracle_mod, s, run, 5)


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_decomposed_fullsize_rigid_vs_oracle(md, oracle_mod, name):
    """The rigid path of the decomposition at full size: c2 (10^6 2CLJQ molecules) and c3
    (5 x 10^5 water molecules) on 4 ranks, their first 10 steps against the oracle (the
    well-conditioned stretch of these runs, tests/test_oracle_sensitivity.py)."""
    s = S.config(name)
    run = md.DecomposedRun(s, 4, transport="loopback")
    compare_run(md, oracle_mod, s, run, 10)


def test_empty_rank_vs_oracle(md, oracle_mod):
    """A rank that owns no molecule: a liquid slab filling x < 0.45 L next to vacuum, two
    boxes cut at 4 of 7 cells -- rank 1 starts with an empty home box (only halo copies of
    the slab's surface) and receives whatever evaporates into it."""
    s0 = S.config("c1s")
    L = s0["box"][0]
    keep = np.nonzero(s0["r"][:, 0] < 0.45 * L)[0]
    s = dict(s0, id=np.arange(len(keep), dtype=np.int64))
    for k in ("r", "v", "q", "j", "comp"):
        s[k] = np.ascontiguousarray(s0[k][keep])
    n = np.floor(np.asarray(s["box"]) / s["rc"]).astype(int)
    boxes = [[0, 0, 0, 4, n[1], n[2]], [4, 0, 0, n[0], n[1], n[2]]]
    run = md.DecomposedRun(s, 2, transport="loopback", boxes=boxes)
    assert run.owned_counts()[1] == 0
    compare_run(md, oracle_mod, s, run, 20)
    assert sum(run.owned_counts()) == len(s["r"])


def test_decomposed_mixture_vs_oracle(md, oracle_mod):
    """Two species with every site kind (LJ, charges, dipoles, quadrupoles; reaction field)
    and the binary parameter eta -- the generic force kernel -- on 2 ranks: the
    component ids travel with the migrants and halo copies, and each rank's N_dof counts
    its species' rotational degrees of freedom."""
    comps = S.random_polar_components()
    s = S.random_system(400, (11.0, 10.0, 12.0), comps, seed_k=101, rc=2.5, eps_rf=4.0)
    eta = np.array([[1.0, 0.9], [0.9, 1.0]])
    run = md.DecomposedRun(s, 2, transport="loopback", eta=eta)
    assert run.lead.get_grid()["kernel"] == 2
    compare_run(md, oracle_mod, s, run, 6, eta=eta)


@pytest.mark.parametrize("name,p", [("c2s", 4), ("c3m", 2)])
def test_rigid_rebalance_vs_oracle(md, oracle_mod, name, p):
    """Rigid molecules (2CLJQ, water) through a rebalance: the run starts from boxes cut
    along z (and y), the k-d tree of the rebalance cuts x first, so every rebalance (every
    4 steps) redistributes molecules -- positions, velocities, quaternions and angular
    momenta travel in the exchange records (k_repartition) -- and every step still
    matches the oracle."""
    s = S.config3(12) if name == "c3m" else S.config(name)
    n = np.floor(np.asarray(s["box"]) / s["rc"]).astype(int)
    if p == 2:
        boxes = [[0, 0, 0, n[0], n[1], 2], [0, 0, 2, n[0], n[1], n[2]]]
    else:
        boxes = [[0, 0, 0, n[0], 2, 2], [0, 2, 0, n[0], n[1], 2], [0, 0, 2, n[0], 2, n[2]],
                 [0, 2, 2, n[0], n[1], n[2]]]
    run = md.DecomposedRun(s, p, transport="loopback", boxes=boxes, rebalance_interval=4)
    compare_run(md, oracle_mod, s, run, 12)
    assert not np.array_equal(np.asarray(run.boxes).reshape(p, 6), np.asarray(boxes))
    assert sum(run.owned_counts()) == len(s["r"])


def test_explicit_rebalance_vs_oracle(md, oracle_mod):
    """mardyn_rebalance mid-run (collective re-partition + redistribution through the
    exchange records) on the slab: the run continues in step with the oracle."""
    s = S.config("c4s")
    run = md.DecomposedRun(s, 8, transport="loopback", boxes=equal_volume_boxes(s, 8))
    run.step(4)
    run.rebalance()
    o = oracle_mod.System(s)
    u0 = o.quantize(s["r"])
    run.step(6)
    hist = run.observable_history(10)
    _, _, _, _, obs = o.run(s["dt"], s["comp"], u0, s["v"], s["q"], s["j"], 10, mode="full")
    for key, ok in (("U_pot", "U"), ("virial", "W"), ("T", "T")):
        assert scaled_err([h[key] for h in hist], obs[ok]).max() <= 1e-5
    assert sorted(run.owned_counts()) != sorted([0] * 8)
    assert sum(run.owned_counts()) == len(s["r"])


def test_nccl_single_rank(md, oracle_mod):
    """mardyn_create_distributed with world = 1: the library's own NCCL communicator
    (dlopen'ed NCCL, ncclCommInitRank) carries the observables (ncclAllGather); the run
    is the one-domain run bit for bit and matches the oracle."""
    s = S.config("c1s")
    uid = md.nccl_unique_id()
    ctx = md.Context.distributed(s["box"], s["rc"], s["components"], s["dt"], uid, 0, 1)
    ctx.partition(s["r"])
    ctx.reserve(len(s["r"]))
    ctx.set_molecules(s["r"], s["v"], comp=s["comp"], q=s["q"], j=s["j"], id=s["id"])
    ctx.step(10)
    h = ctx.get_observable_history(10)
    ref = md.from_system(s)
    ref.step(10)
    assert h == ref.get_observable_history(10)
    o = oracle_mod.System(s)
    _, _, _, _, obs = o.run(s["dt"], s["comp"], o.quantize(s["r"]), s["v"], s["q"], s["j"], 10, mode="full")
    for key, ok in (("U_pot", "U"), ("virial", "W"), ("T", "T")):
        assert scaled_err([x[key] for x in h], obs[ok]).max() <= 1e-5


def test_nvt_decomposed_vs_oracle(md, oracle_mod):
    """NVT velocity rescaling (reading A24) on a decomposed run: the ranks' kinetic
    energies are summed (rank order) before lambda = sqrt(T_target / T(t_k)) is applied,
    so the run follows the oracle's one-domain NVT trajectory."""
    s = S.config("c1s")
    run = md.DecomposedRun(s, 3, transport="loopback")
    run.lead.set_thermostat(1.1, 4)
    run.step(16)
    hist = run.observable_history(16)
    o = oracle_mod.System(s)
    _, _, _, _, obs = o.run(s["dt"], s["comp"], o.quantize(s["r"]), s["v"], s["q"], s["j"], 16, mode="full",
                            T_target=1.1, thermostat_interval=4)
    for key, ok in (("U_pot", "U"), ("virial", "W"), ("T", "T")):
        assert scaled_err([h[key] for h in hist], obs[ok]).max() <= 1e-5, key
    assert abs(hist[4]["T"] - 1.1) < 0.05              # rescaled after step 3
