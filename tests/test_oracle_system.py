"""System-level pins of the oracle (not GPU): pair enumeration, assembly of
site terms into molecular forces / torques / virial, cells, lattice closed
forms, conservation laws."""
import math

import numpy as np
import pytest

import scenarios as S


def lj_shell_sum(a, rc):
    """Closed form for a perfect FCC lattice of LJTS particles (sigma=eps=1):
    U/N = 1/2 sum_shells n_k u(r_k), W/N = 1/2 sum_shells n_k r_k f(r_k),
    enumerating lattice vectors of the FCC lattice directly."""
    rng = range(-4, 5)
    basis = np.array([[0, 0, 0], [.5, .5, 0], [.5, 0, .5], [0, .5, .5]])
    pts = np.array([(i + b[0], j + b[1], k + b[2]) for i in rng for j in rng for k in rng
                    for b in basis]) * a
    r = np.linalg.norm(pts, axis=1)
    r = r[(r > 0) & (r < rc)]
    u = 4 * (r ** -12 - r ** -6) - 4 * (rc ** -12 - rc ** -6)
    w = 24 * (2 * r ** -12 - r ** -6)          # r * f(r)
    return len(r), 0.5 * u.sum(), 0.5 * w.sum()


@pytest.mark.parametrize("n_cells,rho,nb", [(10, 0.6, 42), (8, 0.75, 54)])
def test_fcc_lattice_closed_form(oracle_mod, n_cells, rho, nb):
    """Perfect FCC (configs 0/1 geometry without jitter): every particle has
    the same neighbour count, zero force by inversion symmetry, and U/N, W/N
    equal the shell sums."""
    s = S.lj_fcc(n_cells, rho, 1.0, 0, "lat", 1, jitter=0.0)
    o = oracle_mod.System(s)
    u = o.quantize(s["r"])
    F, _, tot = o.forces(s["comp"], u, s["q"], mode="cells")
    N = len(u)
    a = o.box[0] / n_cells
    nbk, U, W = lj_shell_sum(a, s["rc"])
    assert nbk == nb
    assert tot["npairs"] == N * nb // 2
    assert tot["U"] / N == pytest.approx(U, rel=1e-6)   # lattice snapped to quanta s
    assert tot["W"] / N == pytest.approx(W, rel=1e-6)
    assert np.abs(F).max() < 1e-4


def small_polar_system(n=60, seed_k=100, eps_rf=math.inf):
    comps = S.random_polar_components()
    return S.random_system(n, (7.6, 8.1, 7.9), comps, seed_k=seed_k, rc=2.5, eps_rf=eps_rf)


@pytest.mark.parametrize("eps_rf", [math.inf, 3.0])
def test_three_enumerations_agree(oracle_mod, eps_rf):
    """Brute force O(N^2) minimum image (the definition) == linked-cell
    Newton-3 half shell == full 27-cell shell per molecule, on a
    two-species mixture with every site kind and eta != 1."""
    s = small_polar_system(eps_rf=eps_rf)
    eta = np.array([[1.0, 0.85], [0.85, 1.0]])
    o = oracle_mod.System(s, eta=eta)
    assert min(o.ncell) >= 3
    u = o.quantize(s["r"])
    Fb, tb, Tb = o.forces(s["comp"], u, s["q"], mode="brute")
    Fc, tc, Tc = o.forces(s["comp"], u, s["q"], mode="cells")
    Ff, tf, Tf = o.forces(s["comp"], u, s["q"], mode="full")
    scale = np.abs(Fb).max()
    assert Tb["npairs"] == Tc["npairs"] == Tf["npairs"] > 0
    for X, Y in ((Fb, Fc), (Fb, Ff), (tb, tc), (tb, tf)):
        assert np.abs(X - Y).max() < 1e-11 * scale
    for k in ("U", "W"):
        assert Tb[k] == pytest.approx(Tc[k], rel=1e-11, abs=1e-11)
        assert Tb[k] == pytest.approx(Tf[k], rel=1e-11, abs=1e-11)
    # Newton 3 (Fig. 1): net force vanishes
    assert np.abs(Fb.sum(0)).max() < 1e-11 * scale


def two_molecules(comp, r2, q2, q1=(1, 0, 0, 0), box=40.0, rc=4.0, eps_rf=math.inf):
    s = {"components": [comp], "box": (box,) * 3, "rc": rc, "eps_rf": eps_rf, "lj_shift": 1,
         "comp": np.zeros(2, np.int32)}
    r = np.array([[box / 2] * 3, np.array([box / 2] * 3) + np.asarray(r2, float)])
    q = np.array([q1, q2], float)
    return s, r, q


def qmul(a, b):
    w1, x1, y1, z1 = a; w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


@pytest.mark.parametrize("which", ["c2", "c3", "polarA", "polarB"])
def test_molecular_force_torque_virial_are_gradients(oracle_mod, which):
    """Assembly of site terms into a rigid-molecule pair (reading A1, A6):
    F on molecule 2 = -dU/dr_2 (translation in whole quanta), torque on 2 =
    -dU/dtheta under world-frame rotations of q_2, W = -r_12.F_1, and angular
    momentum balance tau_1 + tau_2 + r_12 x F_2 = 0."""
    comp = {"c2": S.c2_component(), "c3": S.c3_component(),
            "polarA": S.random_polar_components()[0], "polarB": S.random_polar_components()[1]}[which]
    scale_len = 6.0 if which == "c3" else 1.0
    rc = 18.9 if which == "c3" else 4.0
    rng = np.random.default_rng(3)
    q2 = rng.normal(size=4); q2 /= np.linalg.norm(q2)
    q1 = rng.normal(size=4); q1 /= np.linalg.norm(q1)
    r2 = np.array([1.2, 0.3, 0.4]) * scale_len
    s, r, q = two_molecules(comp, r2, q2, q1, box=10 * rc, rc=rc)
    o = oracle_mod.System(s)
    u = o.quantize(r)
    F, tau, tot = o.forces(s["comp"], u, q, mode="brute")
    assert tot["npairs"] == 1
    d = (u[1].astype(np.int64) - u[0].astype(np.int64)) * o.quantum
    scale = max(np.abs(F).max(), np.abs(tau).max())
    K = 64                               # translation by whole quanta
    h = K * o.quantum
    for k in range(3):
        up = u.copy(); up[1, k] += K
        um = u.copy(); um[1, k] -= K
        Up = o.forces(s["comp"], up, q, mode="brute")[2]["U"]
        Um = o.forces(s["comp"], um, q, mode="brute")[2]["U"]
        assert -(Up - Um) / (2 * h) == pytest.approx(F[1, k], abs=2e-6 * scale)
    hr = 1e-5
    for k in range(3):
        n = np.zeros(3); n[k] = 1
        dq = lambda a: np.concatenate([[math.cos(a / 2)], math.sin(a / 2) * n])
        qp = q.copy(); qp[1] = qmul(dq(hr), q[1])
        qm = q.copy(); qm[1] = qmul(dq(-hr), q[1])
        Up = o.forces(s["comp"], u, qp, mode="brute")[2]["U"]
        Um = o.forces(s["comp"], u, qm, mode="brute")[2]["U"]
        assert -(Up - Um) / (2 * hr) == pytest.approx(tau[1, k], abs=2e-6 * scale)
    assert np.abs(F[0] + F[1]).max() < 1e-13 * scale
    assert tot["W"] == pytest.approx(-d @ F[0], rel=1e-12)
    assert np.abs(tau[0] + tau[1] + np.cross(d, F[1])).max() < 1e-11 * scale


def test_quaternion_is_body_to_world(oracle_mod):
    """q = (cos t/2, 0, 0, sin t/2) rotates body x onto world (cos t, sin t, 0):
    a dipole pair built with rotated quaternions has the energy of the same
    world geometry built with identity quaternions and world-frame axes."""
    t = 0.7
    Dx = S.component(1.0, (1, 1, 1), dipoles=[((0, 0, 0), (1, 0, 0), 1.0)])
    Dw = S.component(1.0, (1, 1, 1), dipoles=[((0, 0, 0), (math.cos(t), math.sin(t), 0), 1.0)])
    qz = (math.cos(t / 2), 0, 0, math.sin(t / 2))
    s1, r, q1 = two_molecules(Dx, [2.0, 0.5, 0.3], qz, q1=(1, 0, 0, 0))
    o1 = oracle_mod.System(s1)
    s2, _, q2 = two_molecules(Dw, [2.0, 0.5, 0.3], (1, 0, 0, 0))
    both = {"components": [Dx, Dw], "box": s1["box"], "rc": 4.0}
    o2 = oracle_mod.System(both)
    U1 = o1.forces(np.zeros(2, np.int32), o1.quantize(r), q1, mode="brute")[2]["U"]
    U2 = o2.forces(np.array([0, 1], np.int32), o2.quantize(r), np.array([(1, 0, 0, 0)] * 2, float),
                   mode="brute")[2]["U"]
    assert U1 == pytest.approx(U2, rel=1e-12)


def test_virial_sign_repulsion(oracle_mod):
    """Molecular virial (reading A6) is positive for a repulsive pair."""
    s, r, q = two_molecules(S.lj1_component(), [0.95, 0, 0], (1, 0, 0, 0), rc=2.5)
    o = oracle_mod.System(s)
    F, _, tot = o.forces(s["comp"], o.quantize(r), q, mode="brute")
    assert F[1, 0] > 0 and tot["W"] > 0


def test_cells_definition(oracle_mod):
    """cell_k = floor(x_k n_k / L_k) for positions away from cell faces
    (reading A12), x fastest, counts sum to N."""
    s = S.config0()
    o = oracle_mod.System(s)
    u = o.quantize(s["r"])
    cell, count = o.cells(u)
    x = u * o.quantum
    n = np.array(o.ncell)
    ck = np.floor(x * n / o.box).astype(np.int64)
    frac = x * n / o.box - ck
    safe = np.all((frac > 1e-6) & (frac < 1 - 1e-6), axis=1)
    expect = ck[:, 0] + n[0] * (ck[:, 1] + n[1] * ck[:, 2])
    assert safe.mean() > 0.99
    assert np.array_equal(cell[safe], expect[safe])
    assert count.sum() == len(u)
    assert np.array_equal(np.bincount(cell, minlength=n.prod()), count)


def test_grid_geometry(oracle_mod):
    """n_k = floor(L_k / rc) cells of edge >= rc, quantum a power of
    two with edge <= 2^22 quanta, snapped box within 1e-6 relative."""
    for name in ("c0", "c1s", "c2s", "c3s", "c4s"):
        s = S.config(name)
        o = oracle_mod.System(s)
        L = np.asarray(s["box"])
        assert tuple(o.ncell) == tuple(np.floor(L / s["rc"]).astype(int))
        assert np.all(o.box / np.array(o.ncell) >= s["rc"])
        assert math.log2(o.quantum) == int(math.log2(o.quantum))
        assert np.all(o.edge_q <= 2 ** 22)
        assert np.abs(o.box / L - 1).max() < 1e-6


def test_hit_rate_ideal_gas(oracle_mod):
    """with cells of edge rc only 4 pi/3 / 27 = 15.5 % ("16 %") of the
    27-cell candidates are within rc (homogeneous system)."""
    rng = np.random.default_rng(5)
    L = 25.0
    n = 20000
    s = {"components": [S.lj1_component()], "box": (L,) * 3, "rc": 2.5,
         "comp": np.zeros(n, np.int32)}
    o = oracle_mod.System(s)
    u = o.quantize(rng.uniform(0, L, size=(n, 3)))
    _, count = o.cells(u)
    nc = np.array(o.ncell)
    cnt = count.reshape(nc[2], nc[1], nc[0])
    nb = sum(np.roll(cnt, (dz, dy, dx), axis=(0, 1, 2))
             for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1))
    cand = (cnt * nb).sum() - n
    _, _, tot = o.forces(s["comp"], u, np.tile([1.0, 0, 0, 0], (n, 1)), mode="full")
    ratio = 2 * tot["npairs"] / cand
    edge = o.box[0] / nc[0]
    assert ratio == pytest.approx(4 * math.pi / 3 * 2.5 ** 3 / (27 * edge ** 3), rel=0.02)
    assert edge == pytest.approx(2.5)
    assert ratio == pytest.approx(0.155, abs=0.005)


@pytest.mark.parametrize("shift", [0, 1, -1])
def test_cutoff_boundary_closed_form(oracle_mod, shift):
    """Reading A12 at the cutoff itself: in range iff the exact r^2 < rc^2.  Simple
    cubic lattice of spacing a = rc/2 (8^3 sites): the second axis neighbours sit at
    r = rc exactly and are out; with the x-columns i mod 4 in {0, 1} moved by
    shift = +-1 position quantum, half of the x-axis second neighbours come one
    quantum inside (N/2 more pairs).  Unshifted: every site has 6 + 12 + 8 neighbours
    at a, a sqrt2, a sqrt3, U/N and W/N are the LJTS shell sums, F = 0; brute force
    and linked cells agree."""
    rc = 2.5
    a, n = rc / 2, 8
    idx = np.stack(np.meshgrid(*[np.arange(n)] * 3, indexing="ij"), -1).reshape(-1, 3)
    r = (idx + 0.5) * a
    N = len(r)
    s = S._system("band", (n * a,) * 3, rc, 0.001, 1, 1.0, [S.lj1_component()], r, np.zeros((N, 3)))
    o = oracle_mod.System(s)
    s["r"] = r + np.outer(shift * o.quantum * (idx[:, 0] % 4 < 2), [1.0, 0.0, 0.0])
    u = o.quantize(s["r"])
    assert np.array_equal(u[:, 0].astype(np.int64) - o.quantize(r)[:, 0].astype(np.int64),
                          shift * (idx[:, 0] % 4 < 2))      # exactly one quantum
    res = [o.forces(s["comp"], u, s["q"], mode=m) for m in ("cells", "brute")]
    expect = N * 26 // 2 + (N // 2 if shift else 0)
    for F, _, tot in res:
        assert tot["npairs"] == expect
    if shift == 0:
        d = np.array([1.0] * 6 + [math.sqrt(2)] * 12 + [math.sqrt(3)] * 8) * a
        uu = 4 * (d ** -12 - d ** -6) - 4 * (rc ** -12 - rc ** -6)
        ww = 24 * (2 * d ** -12 - d ** -6)
        F, _, tot = res[0]
        assert tot["U"] / N == pytest.approx(0.5 * uu.sum(), rel=1e-12)
        assert tot["W"] / N == pytest.approx(0.5 * ww.sum(), rel=1e-12)
        assert np.abs(F).max() < 1e-9
    assert res[0][2]["U"] == pytest.approx(res[1][2]["U"], rel=1e-12)
