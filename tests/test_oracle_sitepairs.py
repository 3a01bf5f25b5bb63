"""Pins of the oracle's site-site kernels (not GPU).

Each pin is something the paper or mathematics fixes independently of the
oracle's formulas:
  * LJ 12-6 (Eq. 1): minimum U = -eps at r = 2^(1/6) sigma
    with zero force, zero crossing at sigma, SPEC S:153 value at 2.5 sigma;
  * LJTS (reading A2): U(rc) = 0, shifted value at r = 1;
  * multipoles (reading A5): every closed form equals the
    point-charge limit of its charge representation (Richardson-extrapolated),
    for energy, force and torque;
  * every kernel: force = -gradient (central differences), torque = minus the
    derivative under rotation, angular-momentum balance per pair;
  * reaction field (reading A4): eps_RF = 1 limit, eps_RF = inf zero force
    and energy at rc, the mu-mu correction value of SPEC S:197.
"""
import math

import numpy as np
import pytest

LJ, CH, DI, QU = 0, 1, 2, 3


def make_sys(oracle_mod, rc=2.5, eps_rf=math.inf, lj_shift=1):
    import scenarios as S
    sys_d = {"components": [S.lj1_component()], "box": (10 * rc,) * 3, "rc": rc,
             "eps_rf": eps_rf, "lj_shift": lj_shift}
    return oracle_mod.System(sys_d)


def site(oracle_mod, kind, m=1.0, sigma=1.0, eps=1.0):
    return oracle_mod.make_site(kind, (0, 0, 0), (0, 0, 1), m, sigma, eps)


def unit(v):
    v = np.asarray(v, dtype=np.float64)
    return v / np.linalg.norm(v)


# --------------------------------------------------------------------------- LJ

def test_lj_minimum_zero_crossing_and_value(oracle_mod):
    o = make_sys(oracle_mod, lj_shift=0)
    a = site(oracle_mod, LJ)
    rmin = 2 ** (1 / 6)
    u, fb, _, _ = o.site_pair(a, [0, 0, 1], a, [0, 0, 1], [rmin, 0, 0])
    assert u == pytest.approx(-1.0, abs=1e-14)           # P:72 minimum -eps
    assert np.abs(fb).max() < 1e-13                       # dU/dr = 0 there
    u, _, _, _ = o.site_pair(a, [0, 0, 1], a, [0, 0, 1], [0, 1.0, 0])
    assert u == pytest.approx(0.0, abs=1e-15)             # U(sigma) = 0
    u, _, _, _ = o.site_pair(a, [0, 0, 1], a, [0, 0, 1], [0, 0, 2.5])
    assert u == pytest.approx(-1.6316891136e-2, rel=1e-10)


def test_ljts_shift(oracle_mod):
    o = make_sys(oracle_mod, lj_shift=1)
    a = site(oracle_mod, LJ)
    u, _, _, _ = o.site_pair(a, [0, 0, 1], a, [0, 0, 1], [1.0, 0, 0])
    assert u == pytest.approx(1.6316891136e-2, rel=1e-10)
    u, fb, _, _ = o.site_pair(a, [0, 0, 1], a, [0, 0, 1], [2.5 * (1 - 1e-12), 0, 0])
    assert abs(u) < 1e-12                                    # continuous at rc
    # force is not shifted: jump of |F| at rc (attractive side), reading A2
    assert fb[0] == pytest.approx(-0.0389995, rel=1e-5)


def test_lorentz_berthelot_eta(oracle_mod):
    """P:77 combination rules on an unlike pair (SPEC S:165 examples):
    sigma 1|3 -> 2, eps 4|9 -> 6 (eta=1) and 3 (eta=0.5).  Checked through the
    energy zero (r = sigma_ab) and the minimum value (-eps_ab)."""
    o = make_sys(oracle_mod, rc=20.0, lj_shift=0)
    a = oracle_mod.make_site(LJ, (0, 0, 0), sigma=1.0, eps=4.0)
    b = oracle_mod.make_site(LJ, (0, 0, 0), sigma=3.0, eps=9.0)
    z = [0, 0, 1]
    u, _, _, _ = o.site_pair(a, z, b, z, [2.0, 0, 0])
    assert abs(u) < 1e-13
    u, _, _, _ = o.site_pair(a, z, b, z, [2.0 * 2 ** (1 / 6), 0, 0])
    assert u == pytest.approx(-6.0, rel=1e-13)
    u, _, _, _ = o.site_pair(a, z, b, z, [2.0 * 2 ** (1 / 6), 0, 0], eta=0.5)
    assert u == pytest.approx(-3.0, rel=1e-13)


# ----------------------------------------------------------------- multipoles

def charge_rep(kind, m, pos, axis, d):
    """Point charges representing a point multipole of moment m (reading A5):
    dipole mu = q d (charges +-q at +-d/2); linear quadrupole Q = sum q z^2 =
    2 q d^2 (q at +-d, -2q at the centre)."""
    pos = np.asarray(pos, float); axis = unit(axis)
    if kind == CH:
        return [(pos, m)]
    if kind == DI:
        q = m / d
        return [(pos + 0.5 * d * axis, q), (pos - 0.5 * d * axis, -q)]
    if kind == QU:
        q = m / (2 * d * d)
        return [(pos + d * axis, q), (pos - d * axis, q), (pos, -2 * q)]
    raise ValueError


def charges_pair(o, oracle_mod, ka, ma, ea, kb, mb, eb, rv, d):
    """Energy, force on b (total) and torques about each site from the
    charge representations, using only the oracle's charge-charge kernel
    with eps_RF = 1 (plain Coulomb up to a constant that cancels for neutral
    multipoles)."""
    A = charge_rep(ka, ma, [0, 0, 0], ea, d)
    B = charge_rep(kb, mb, rv, eb, d)
    U = 0.0; Fb = np.zeros(3); ta = np.zeros(3); tb = np.zeros(3)
    for pa, qa in A:
        for pb, qb in B:
            sa = oracle_mod.make_site(CH, (0, 0, 0), m=qa)
            sb = oracle_mod.make_site(CH, (0, 0, 0), m=qb)
            u, f, _, _ = o.site_pair(sa, [0, 0, 1], sb, [0, 0, 1], np.asarray(pb) - pa)
            U += u; Fb += f
            tb += np.cross(np.asarray(pb) - rv, f)
            ta += np.cross(pa, -f)
    return U, Fb, ta, tb


KINDS = [(CH, DI), (DI, CH), (CH, QU), (QU, CH), (DI, DI), (DI, QU), (QU, DI), (QU, QU)]
SCALE_POW = {(CH, DI): 2, (CH, QU): 3, (DI, DI): 3, (DI, QU): 4, (QU, QU): 5}


@pytest.mark.parametrize("ka,kb", KINDS)
def test_multipole_point_charge_limit(oracle_mod, ka, kb):
    """Closed forms = Richardson-extrapolated point-charge limit, for U, f_b,
    tau_a, tau_b, on random geometries (error normalised by the natural
    scale m_a m_b / r^p)."""
    o = make_sys(oracle_mod, rc=50.0, eps_rf=1.0)
    rng = np.random.default_rng(7 + 10 * ka + kb)
    ma, mb = 0.7, 1.3
    p = SCALE_POW[tuple(sorted((ka, kb)))]
    for _ in range(5):
        ea, eb = unit(rng.normal(size=3)), unit(rng.normal(size=3))
        r = 1.5 + rng.uniform()
        rv = unit(rng.normal(size=3)) * r
        sa = oracle_mod.make_site(ka, (0, 0, 0), ea, ma)
        sb = oracle_mod.make_site(kb, (0, 0, 0), eb, mb)
        u, fb, ta, tb = o.site_pair(sa, ea, sb, eb, rv)
        d = 1e-2 * r
        U1, F1, ta1, tb1 = charges_pair(o, oracle_mod, ka, ma, ea, kb, mb, eb, rv, d)
        U2, F2, ta2, tb2 = charges_pair(o, oracle_mod, ka, ma, ea, kb, mb, eb, rv, d / 2)
        ext = lambda x1, x2: (4 * x2 - x1) / 3
        scale = ma * mb / r ** p
        assert abs(u - ext(U1, U2)) < 2e-6 * scale
        assert np.abs(fb - ext(F1, F2)).max() < 2e-6 * scale / r
        assert np.abs(ta - ext(ta1, ta2)).max() < 2e-6 * scale
        assert np.abs(tb - ext(tb1, tb2)).max() < 2e-6 * scale


def test_multipole_fixed_orientation_values(oracle_mod):
    """Special cases that reduce to textbook values (SPEC S:178 head-to-tail
    dipoles -2 mu^2/r^3; collinear quadrupoles 6 Q^2/r^5; T-shape -3;
    mu and Q along r: 3 mu Q / r^4)."""
    o = make_sys(oracle_mod, rc=50.0, eps_rf=1.0)
    x = [1, 0, 0]; y = [0, 1, 0]
    D = oracle_mod.make_site(DI, (0, 0, 0), x, 1.0)
    Q = oracle_mod.make_site(QU, (0, 0, 0), x, 1.0)
    u, *_ = o.site_pair(D, x, D, x, [2.0, 0, 0]); assert u == pytest.approx(-0.25, rel=1e-13)
    u, *_ = o.site_pair(D, y, D, y, [2.0, 0, 0]); assert u == pytest.approx(0.125, rel=1e-13)
    u, *_ = o.site_pair(Q, x, Q, x, [1.0, 0, 0]); assert u == pytest.approx(6.0, rel=1e-13)
    u, *_ = o.site_pair(Q, x, Q, y, [1.0, 0, 0]); assert u == pytest.approx(-3.0, rel=1e-13)
    u, *_ = o.site_pair(Q, y, Q, y, [1.0, 0, 0]); assert u == pytest.approx(2.25, rel=1e-13)
    u, *_ = o.site_pair(D, x, Q, x, [1.0, 0, 0]); assert u == pytest.approx(3.0, rel=1e-13)


# ----------------------------------------------------- gradient consistency

ALL = [(LJ, LJ), (CH, CH)] + KINDS


def rot(v, n, h):
    """Rodrigues rotation of v about unit n by angle h."""
    v = np.asarray(v, float)
    return v * math.cos(h) + np.cross(n, v) * math.sin(h) + n * (n @ v) * (1 - math.cos(h))


@pytest.mark.parametrize("ka,kb", ALL)
@pytest.mark.parametrize("eps_rf", [1.0, 7.5, math.inf])
def test_force_torque_are_gradients(oracle_mod, ka, kb, eps_rf):
    o = make_sys(oracle_mod, rc=3.0, eps_rf=eps_rf)
    rng = np.random.default_rng(11 + 10 * ka + kb)
    for _ in range(4):
        ea, eb = unit(rng.normal(size=3)), unit(rng.normal(size=3))
        rv = unit(rng.normal(size=3)) * (1.0 + rng.uniform())
        sa = oracle_mod.make_site(ka, (0, 0, 0), ea, 0.8, 1.0, 1.0)
        sb = oracle_mod.make_site(kb, (0, 0, 0), eb, 1.1, 1.0, 1.0)
        u, fb, ta, tb = o.site_pair(sa, ea, sb, eb, rv)
        h = 1e-6
        scale = max(1.0, np.abs(fb).max(), np.abs(ta).max(), np.abs(tb).max())
        for k in range(3):
            dv = np.zeros(3); dv[k] = h
            up = o.site_pair(sa, ea, sb, eb, rv + dv)[0]
            um = o.site_pair(sa, ea, sb, eb, rv - dv)[0]
            assert -(up - um) / (2 * h) == pytest.approx(fb[k], abs=1e-6 * scale)
        for k in range(3):
            n = np.zeros(3); n[k] = 1.0
            up = o.site_pair(sa, rot(ea, n, h), sb, eb, rv)[0]
            um = o.site_pair(sa, rot(ea, n, -h), sb, eb, rv)[0]
            assert -(up - um) / (2 * h) == pytest.approx(ta[k], abs=1e-6 * scale)
            up = o.site_pair(sa, ea, sb, rot(eb, n, h), rv)[0]
            um = o.site_pair(sa, ea, sb, rot(eb, n, -h), rv)[0]
            assert -(up - um) / (2 * h) == pytest.approx(tb[k], abs=1e-6 * scale)
        # angular-momentum balance of one site pair: ta + tb + r x f_b = 0
        assert np.abs(ta + tb + np.cross(rv, fb)).max() < 1e-12 * scale


# ----------------------------------------------------------- reaction field

def test_reaction_field_limits(oracle_mod):
    rc = 2.5
    q1 = oracle_mod.make_site(CH, (0, 0, 0), m=1.0)
    q2 = oracle_mod.make_site(CH, (0, 0, 0), m=-1.0)
    z = [0, 0, 1]
    # eps_RF = 1: plain Coulomb shifted by a constant
    o1 = make_sys(oracle_mod, rc=rc, eps_rf=1.0)
    u, fb, _, _ = o1.site_pair(q1, z, q2, z, [2.0, 0, 0])
    assert u == pytest.approx(-1 / 2.0 + 1 / rc, rel=1e-14)
    assert fb[0] == pytest.approx(-1 / 4.0, rel=1e-14)         # b pulled towards a
    # conducting boundary: energy and force vanish at rc
    oi = make_sys(oracle_mod, rc=rc, eps_rf=math.inf)
    u, fb, _, _ = oi.site_pair(q1, z, q2, z, [rc, 0, 0])
    assert abs(u) < 1e-15 and np.abs(fb).max() < 1e-15
    # mu-mu RF term: parallel dipoles, mu = 1, rc = 2.5: -1/rc^3 = -0.064
    D = oracle_mod.make_site(DI, (0, 0, 0), z, 1.0)
    u_inf = oi.site_pair(D, z, D, z, [1.0, 0, 0])[0]
    u_one = o1.site_pair(D, z, D, z, [1.0, 0, 0])[0]
    assert u_inf - u_one == pytest.approx(-0.064, rel=1e-13)
