"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on
the same seeded inputs.  Small configs are compared element
by element; they span several cell tiles, ragged cells, empty cells and the
chunked paths of the force kernels."""
import math

import numpy as np
import pytest

import scenarios as S
from parity_util import (assert_forces_close, assert_rel, candidates_from_counts, min_image, rms)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def md():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1408_4599_b200 import build, mardyn
    build.build()
    return mardyn


def gpu_state(md, s, eta=None):
    ctx = md.from_system(s, eta=eta)
    F, tau = ctx.get_forces()               # F(t0), tau(t0) from set_molecules (A8)
    ctx.compute_forces()
    obs = ctx.get_observables()
    u, cell, count = ctx.get_raw()
    return ctx, F, tau, obs, u, cell, count


def oracle_state(oracle_mod, s, eta=None, mode="full"):
    o = oracle_mod.System(s, eta=eta)
    u = o.quantize(s["r"])
    cell, count = o.cells(u)
    F, tau, tot = o.forces(s["comp"], u, s["q"], mode=mode)
    return o, u, cell, count, F, tau, tot


def check_step0(md, oracle_mod, s, eta=None, torque=True):
    ctx, Fg, tg, obs, ug, cg, ng = gpu_state(md, s, eta)
    o, uo, co, no, Fo, to, tot = oracle_state(oracle_mod, s, eta)
    g = ctx.get_grid()
    assert tuple(g["ncell"]) == tuple(o.ncell)
    assert g["quantum"] == o.quantum
    assert np.array_equal(np.array(g["period"]), o.period)
    # bit-exact lattice, cells, counts (north_star)
    assert np.array_equal(ug, uo)
    assert np.array_equal(cg, co)
    assert np.array_equal(ng, no)
    assert obs["n_pairs"] == tot["npairs"]
    assert obs["n_candidates"] == candidates_from_counts(no, o.ncell)
    assert_forces_close(Fg, Fo, "force")
    if torque:
        assert_forces_close(tg, to, "torque")
    assert_rel(obs["U_pot"], tot["U"], "U_pot")
    assert_rel(obs["virial"], tot["W"], "virial")
    return ctx, o


@pytest.mark.parametrize("name", ["c0", "c1s", "c4s"])
def test_step0_lj(md, oracle_mod, name):
    check_step0(md, oracle_mod, S.config(name), torque=False)


@pytest.mark.parametrize("name", ["c2s", "c3s"])
def test_step0_rigid(md, oracle_mod, name):
    check_step0(md, oracle_mod, S.config(name))


@pytest.mark.parametrize("eps_rf", [math.inf, 4.0])
def test_step0_generic_mixture(md, oracle_mod, eps_rf):
    """Two species, every site kind (LJ, charges, dipoles, quadrupoles),
    unlike-pair binary parameter eta: generic kernel."""
    comps = S.random_polar_components()
    s = S.random_system(400, (11.0, 10.0, 12.0), comps, seed_k=101, rc=2.5, eps_rf=eps_rf)
    eta = np.array([[1.0, 0.9], [0.9, 1.0]])
    ctx, _ = check_step0(md, oracle_mod, s, eta=eta)
    assert ctx.get_grid()["kernel"] == 2


def test_dense_cells_chunking(md, oracle_mod):
    """~77 molecules per cell: i-chunks of 32 and neighbourhoods larger than
    the shared-memory slab (chunked staging) in both kernels."""
    s = S.lj_fcc(9, 1.2, 1.0, 7, "dense", 1, jitter=0.02, rc=4.0)
    check_step0(md, oracle_mod, s, torque=False)
    comp = S.c2_component()
    s2 = S.lj_fcc(6, 0.9, 1.0, 8, "dense2", 1, jitter=0.0, rc=3.2)
    rng = np.random.default_rng(3)
    s2["components"] = [comp]
    s2["q"] = S.random_quaternions(rng, len(s2["r"]))
    s2["j"] = S.angular_momenta(rng, s2["q"], comp["inertia"], 1.0)
    check_step0(md, oracle_mod, s2)


@pytest.mark.parametrize("comp_name", ["c2", "c3"])
def test_dense_rigid_batches_and_chunks(md, oracle_mod, comp_name):
    """k_force_rigid3 beyond its common case: ~76 molecules per cell (home
    molecules in batches of 64) and 27-cell neighbourhoods of 2048 molecules
    (staged in chunks of 1152), 2CLJQ and TIP4P shapes."""
    s = S.lj_fcc(8, 0.9, 1.0, 9, "dense3", 1, jitter=0.01, rc=4.3)
    rng = np.random.default_rng(4)
    if comp_name == "c2":
        comp = S.c2_component()
    else:
        # TIP4P-like shape in reduced units: the config-3 site geometry scaled to ~0.3 sigma,
        # charges +0.3, +0.3, -0.6 on H, H, M, one LJ site (sigma = eps = 1)
        tip = S.config("c3s")["components"][0]
        k = 0.3 / 1.43
        comp = dict(tip)
        comp["lj"] = [(tuple(k * x for x in p_), 1.0, 1.0) for p_, _, _ in tip["lj"]]
        comp["charges"] = [(tuple(k * x for x in p_), 0.3 if q > 0 else -0.6) for p_, q in tip["charges"]]
        comp["mass"] = 1.0
        comp["inertia"] = (0.02, 0.05, 0.03)
        s["eps_rf"] = math.inf
    s["components"] = [comp]
    s["q"] = S.random_quaternions(rng, len(s["r"]))
    s["j"] = S.angular_momenta(rng, s["q"], comp["inertia"], 1.0)
    ctx, _ = check_step0(md, oracle_mod, s)
    assert ctx.get_grid()["kernel"] == 1


@pytest.mark.parametrize("n_cells,rho,rc", [(5, 0.75, 2.5), (6, 0.75, 2.5), (7, 0.8, 2.5), (6, 0.9, 1.6)])
def test_step0_lj_boxes(md, oracle_mod, n_cells, rho, rc):
    """Single-site kernel on small boxes (3-6 cells per axis: sub-chunks
    limited to nx - 2 cells, periodic wrap pieces in every staged row)."""
    s = S.lj_fcc(n_cells, rho, 1.0, 40 + n_cells, f"box{n_cells}", 1, jitter=0.05, rc=rc)
    check_step0(md, oracle_mod, s, torque=False)


@pytest.mark.parametrize("n,box", [(700, (30.0, 30.0, 30.0)), (1500, (60.0, 25.0, 20.0))])
def test_step0_lj_gas(md, oracle_mod, n, box):
    """Gases (0.2-0.5 molecules per cell): blocks of 32 molecules spanning
    many cells and rows take the per-lane path."""
    s = S.random_system(n, box, [S.lj1_component()], seed_k=120 + n, rc=2.5, dmin=1.0)
    check_step0(md, oracle_mod, s, torque=False)


def run_both(md, oracle_mod, s, nsteps, eta=None):
    ctx = md.from_system(s, eta=eta)
    ctx.step(nsteps)
    hist = ctx.get_observable_history(nsteps)
    mol = ctx.get_molecules()
    o = oracle_mod.System(s, eta=eta)
    u, v, q, j, obs = o.run(s["dt"], s["comp"], o.quantize(s["r"]), s["v"], s["q"], s["j"], nsteps,
                            half_step=0, mode="full")
    return ctx, hist, mol, o, u, v, q, j, obs


@pytest.mark.parametrize("name,nsteps", [("c0", 10), ("c1s", 20), ("c2s", 10), ("c3s", 10), ("c4s", 10)])
def test_trajectory(md, oracle_mod, name, nsteps):
    """Independent GPU / oracle trajectories from the same initial state:
    per-step U, W, T within 1e-5 relative, positions within 1e-4 sigma."""
    s = S.config(name)
    ctx, hist, mol, o, u, v, q, j, obs = run_both(md, oracle_mod, s, nsteps)
    assert len(hist) == nsteps
    for k in range(nsteps):
        assert hist[k]["step"] == k
        assert hist[k]["n_pairs"] == obs["npairs"][k]
        assert_rel(hist[k]["U_pot"], obs["U"][k], f"U[{k}]")
        assert_rel(hist[k]["virial"], obs["W"][k], f"W[{k}]")
        assert_rel(hist[k]["T"], obs["T"][k], f"T[{k}]")
    box = o.box
    d = min_image(mol["r"] - u * o.quantum, box)
    sigma = s["components"][0]["lj"][0][1]
    assert np.abs(d).max() <= 1e-4 * sigma
    if name in ("c2s", "c3s"):
        dq = np.minimum(np.abs(mol["q"] - q).max(1), np.abs(mol["q"] + q).max(1))
        assert dq.max() < 1e-4


@pytest.mark.parametrize("variant", ["sym", "sym_pc_only", "generic", "sym_unequal_h", "pc_off_axis_lj",
                                     "generic_off_centre_q"])
def test_2cljq_kernel_instances(md, oracle_mod, monkeypatch, variant):
    """The three instances of the 2CLJQ force kernel against the oracle: the
    linear-molecule one (c2's molecule, and LJ sites at unequal distances on the axis), the
    polar-at-COM one (MARDYN_NO_SYM=1, or an LJ site off the axis), and the generic one
    (MARDYN_NO_POLAR_COM=1, or the quadrupole off the centre of mass).  F(t0), tau(t0), U, W,
    cells bit-exact, then 8 steps of U, W, T, positions and orientations."""
    s = dict(S.config("c2s"))
    c = dict(s["components"][0])
    qm = c["quadrupoles"][0][2]
    if variant == "sym_pc_only":
        monkeypatch.setenv("MARDYN_NO_SYM", "1")
    elif variant == "generic":
        monkeypatch.setenv("MARDYN_NO_POLAR_COM", "1")
    elif variant == "sym_unequal_h":
        c["lj"] = [((0.0, 0.0, 0.3), 1.0, 1.0), ((0.0, 0.0, -0.2), 1.0, 1.0)]
    elif variant == "pc_off_axis_lj":
        c["lj"] = [((0.05, 0.0, 0.25), 1.0, 1.0), ((0.0, 0.0, -0.25), 1.0, 1.0)]
    elif variant == "generic_off_centre_q":
        c["quadrupoles"] = [((0.0, 0.0, 0.1), (0.0, 0.0, 1.0), qm)]
    s["components"] = [c]
    check_step0(md, oracle_mod, s)
    nsteps = 8
    ctx, hist, mol, o, u, v, q, j, obs = run_both(md, oracle_mod, s, nsteps)
    for k in range(nsteps):
        assert hist[k]["n_pairs"] == obs["npairs"][k]
        assert_rel(hist[k]["U_pot"], obs["U"][k], f"U[{k}]")
        assert_rel(hist[k]["virial"], obs["W"][k], f"W[{k}]")
        assert_rel(hist[k]["T"], obs["T"][k], f"T[{k}]")
    assert np.abs(min_image(mol["r"] - u * o.quantum, o.box)).max() <= 1e-4
    dq = np.minimum(np.abs(mol["q"] - q).max(1), np.abs(mol["q"] + q).max(1))
    assert dq.max() < 1e-4


@pytest.mark.parametrize("name,nsteps", [("c2s", 60), ("c3s", 60)])
def test_rigid_long_run(md, oracle_mod, name, nsteps):
    """Longer rigid-body runs (Fincham rotation, reading A7).  Independent fp32 and
    fp64 trajectories part chaotically (c2s starts from close random-orientation
    contacts), so the per-step protocol is a snapshot: after the run the oracle
    evaluates the GPU's own state (positions, quaternions) -- forces and torques
    within A15, U and W within 1e-5 -- and the GPU conserves total energy as well
    as the oracle's own trajectory does (its drift + 1e-5 of the kinetic energy)."""
    s = S.config(name)
    ctx, hist, mol, o, u, v, q, j, obs = run_both(md, oracle_mod, s, nsteps)
    Eg = np.array([x["U_pot"] + x["E_kin_trans"] + x["E_kin_rot"] for x in hist])
    ekin = np.array([x["E_kin_trans"] + x["E_kin_rot"] for x in hist])
    Eo = np.asarray(obs["U"]) + np.asarray(obs["KEt"]) + np.asarray(obs["KEr"])
    drift, drift_o = np.abs(Eg - Eg[0]).max(), np.abs(Eo - Eo[0]).max()
    assert drift <= drift_o + 1e-5 * ekin.mean(), (drift, drift_o)
    # snapshot parity on the GPU's state at t_n
    ctx.compute_forces()
    og = ctx.get_observables()
    Fg, tg = ctx.get_forces()
    ug, _, _ = ctx.get_raw()
    m = ctx.get_molecules()
    Fo, to, tot = o.forces(s["comp"], ug, m["q"], mode="full")
    assert og["n_pairs"] == tot["npairs"]
    assert_forces_close(Fg, Fo, "force")
    assert_forces_close(tg, to, "torque")
    assert_rel(og["U_pot"], tot["U"], "U_pot")
    assert_rel(og["virial"], tot["W"], "virial")


def test_initial_temperature_and_nve(md):
    """A8 pin on the GPU: T(0) = generator T; NVE over 400 steps of config 0
    within 2.5e-4 eps per particle (the oracle's own bound)."""
    s = S.config0()
    ctx = md.from_system(s)
    ctx.step(400)
    h = ctx.get_observable_history(400)
    assert h[0]["T"] == pytest.approx(s["T"], rel=1e-5)
    E = np.array([x["U_pot"] + x["E_kin_trans"] + x["E_kin_rot"] for x in h])
    assert np.abs(E - E[0]).max() / len(s["r"]) < 2.5e-4


def test_determinism(md):
    """Canonical in-cell order + fixed-order sums: two runs agree bitwise."""
    s = S.config("c1s")
    out = []
    for _ in range(2):
        ctx = md.from_system(s)
        ctx.step(15)
        m = ctx.get_molecules()
        out.append((m["r"].copy(), m["v"].copy(), ctx.get_observables()))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]


def test_determinism_rigid(md):
    """The load-balanced rigid kernel (ballot-compacted partner lists, fixed-order
    group reductions, slice partials summed in order): bitwise identical reruns."""
    s = S.config("c3s")
    out = []
    for _ in range(2):
        ctx = md.from_system(s)
        ctx.step(8)
        m = ctx.get_molecules()
        F, tau = ctx.get_forces()
        out.append((m["r"].copy(), m["q"].copy(), m["j"].copy(), F.copy(), tau.copy(), ctx.get_observables()))
    for a, b in zip(out[0], out[1]):
        if isinstance(a, dict):
            assert a == b
        else:
            assert np.array_equal(a, b)


def test_determinism_decomposed_async(md):
    """Decomposed run, asynchronous exchange (records packed in arrival order,
    imported, then sorted canonically): bitwise identical reruns."""
    s = S.config("c1s")
    out = []
    for _ in range(2):
        run = md.DecomposedRun(s, 2, transport="loopback")
        run.step(6)
        m = run.molecules()
        out.append((m["r"].copy(), m["v"].copy(), run.observables()))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]


def test_errors(md):
    s = S.config0()
    with pytest.raises(md.MardynError) as e:
        md.Context((5.0, 5.0, 5.0), 2.5, s["components"], 0.002)
    assert e.value.code == -1
    ctx = md.Context(s["box"], 2.5, s["components"], 0.002)
    with pytest.raises(md.MardynError) as e:
        ctx.step(1)
    assert e.value.code == -7
    r = s["r"].copy()
    r[17, 1] = np.nan                             # invalid input: validated on the device
    with pytest.raises(md.MardynError) as e:
        ctx.set_molecules(r, s["v"], comp=s["comp"], half_step=1)
    assert e.value.code == -1
    comp = s["comp"].copy()
    comp[5] = 3
    with pytest.raises(md.MardynError) as e:
        ctx.set_molecules(s["r"], s["v"], comp=comp, half_step=1)
    assert e.value.code == -1
    v = s["v"].copy()
    v[0] = [1e5, 0, 0]
    ctx.set_molecules(s["r"], v, comp=s["comp"], half_step=1)
    ctx.step(1)
    with pytest.raises(md.MardynError) as e:
        ctx.get_observables()
    assert e.value.code == -3


def test_nvt_trajectory_and_tail(md, oracle_mod):
    """NVT velocity rescaling (reading A24) toward T = 1.2 every 5 steps:
    per-step U, W, T and final positions match the oracle's NVT run; the
    tail corrections of the loaded system match the oracle's."""
    s = S.config0()
    nsteps = 20
    ctx = md.from_system(s)
    ctx.set_thermostat(1.2, 5)
    ctx.step(nsteps)
    hist = ctx.get_observable_history(nsteps)
    mol = ctx.get_molecules()
    o = oracle_mod.System(s)
    u, v, q, j, obs = o.run(s["dt"], s["comp"], o.quantize(s["r"]), s["v"], s["q"], s["j"], nsteps,
                            half_step=0, mode="full", T_target=1.2, thermostat_interval=5)
    for k in range(nsteps):
        assert hist[k]["n_pairs"] == obs["npairs"][k]
        for key, ok in (("U_pot", "U"), ("virial", "W"), ("T", "T")):
            assert_rel(hist[k][key], obs[ok][k], f"{key}[{k}]")
    assert abs(hist[-1]["T"] - 1.2) < 0.1
    d = min_image(mol["r"] - u * o.quantum, o.box)
    assert np.abs(d).max() <= 1e-4
    U, W = ctx.get_tail_corrections()
    Uo, Wo = o.lj_tail([len(s["r"])], float(np.prod(o.box)))
    assert U == pytest.approx(Uo, rel=1e-12) and W == pytest.approx(Wo, rel=1e-12)
    with pytest.raises(md.MardynError):
        ctx.set_thermostat(-1.0, 5)


@pytest.mark.parametrize("which", ["clj2q", "tip4p"])
def test_rigid_pair_golden_gpu(md, which):
    """The CUDA path on the SURVEY 8(c) pair pins (two molecules: rigid kernel,
    quaternion convention, lever-arm torque, reaction field, virial sign) --
    fp32 against the printed 8-digit values."""
    from test_golden import pair_system
    s, g = pair_system(which)
    ctx = md.from_system(s)
    F, tau = ctx.get_forces()
    ctx.compute_forces()
    obs = ctx.get_observables()
    assert ctx.get_grid()["kernel"] == 1
    assert obs["n_pairs"] == 1
    assert_rel(obs["U_pot"], g["U"], "U_pot", tol=5e-5)
    assert_rel(obs["virial"], g["W"], "virial", tol=5e-5)
    scale = np.abs(g["F2"]).max()
    assert np.abs(F[1] - g["F2"]).max() <= 5e-5 * scale, (F[1], g["F2"])
    assert np.abs(tau[1] - g["tau2"]).max() <= 5e-5 * np.abs(g["tau2"]).max(), (tau[1], g["tau2"])


@pytest.mark.parametrize("model", ["lj", "2cljq"])
@pytest.mark.parametrize("shift", [0, 1, -1])
def test_guard_band_exact(md, oracle_mod, model, shift):
    """Pairs exactly at the cutoff and one position quantum inside / outside it
    (reading A12: in range iff the exact r^2 < rc^2, decided in integer quanta).
    Simple cubic lattice of spacing rc/2: the second axis neighbours sit at r = rc
    exactly, so the fp32 fast passes of both force kernels see them in the guard band
    and the exact pass decides them.  shift = +-1: the molecules of x-columns
    i mod 4 in {0, 1} move by +-1 quantum along x, so half of the x-axis second
    neighbours come one quantum inside rc.  n_pairs is pinned in closed form
    (26 neighbours with r^2 / a^2 in {1, 2, 3} per molecule, + N/2 for the shifted
    lattice) and forces / U / W against the oracle."""
    rc = 2.5 if model == "lj" else 4.0
    a, n = rc / 2, 8
    idx = np.stack(np.meshgrid(*[np.arange(n)] * 3, indexing="ij"), -1).reshape(-1, 3)
    r = (idx + 0.5) * a
    N = len(r)
    rng = np.random.default_rng(77)
    if model == "lj":
        comps, q = [S.lj1_component()], None
    else:
        comps, q = [S.c2_component()], S.random_quaternions(rng, N)
    s = S._system(f"band_{model}", (n * a,) * 3, rc, 0.001, 1, 1.0, comps, r, np.zeros((N, 3)), q=q)
    quantum = oracle_mod.System(s).quantum
    s["r"] = np.ascontiguousarray(r + np.outer(shift * quantum * (idx[:, 0] % 4 < 2), [1.0, 0.0, 0.0]))
    ctx, Fg, tg, obs, ug, cg, ng = gpu_state(md, s)
    o, uo, co, no, Fo, to, tot = oracle_state(oracle_mod, s)
    assert np.array_equal(ug, uo) and np.array_equal(cg, co) and np.array_equal(ng, no)
    expect = N * 26 // 2 + (N // 2 if shift else 0)
    assert tot["npairs"] == expect
    assert obs["n_pairs"] == expect
    assert_rel(obs["U_pot"], tot["U"], "U_pot")
    assert_rel(obs["virial"], tot["W"], "virial")
    # the LJ lattice is (nearly) force-free by symmetry: the force tolerance is taken
    # relative to the nearest-neighbour pair force instead of the RMS molecular force
    scale = max(rms(Fo), abs(24 * (2 * a ** -13 - a ** -7)))
    assert np.abs(Fg - Fo).max() <= 1e-4 * scale
    if model != "lj":
        assert_forces_close(tg, to, "torque")
