"""Pins of the oracle's integrator (not GPU): leapfrog Eqs. 2-3 (PAPER.md
P:163-171) and the Fincham quaternion leapfrog reading of Eqs. 4-5 (P:172-180,
reading A7), with the A8 start and A9 temperature."""
import math

import numpy as np
import pytest

import scenarios as S


def lone(comp, box=40.0, rc=4.0, v=(0, 0, 0), q=(1, 0, 0, 0), j=(0, 0, 0)):
    s = {"components": [comp], "box": (box,) * 3, "rc": rc}
    return s, np.zeros(1, np.int32), np.array([[box / 2] * 3]), np.array([v], float), \
        np.array([q], float), np.array([j], float)


def test_free_flight_exact(oracle_mod):
    """F = 0: r(t+dt) = r(t) + dt v exactly on the position lattice."""
    s, comp, r, v, q, j = lone(S.lj1_component(), v=(0.3, -1.7, 2.2))
    o = oracle_mod.System(s)
    u0 = o.quantize(r)
    dt = 0.002
    u, v1, _, _, obs = o.run(dt, comp, u0, v, q, j, 25, half_step=1, mode="brute")
    step = np.rint(dt * v[0] / o.quantum).astype(np.int64)
    assert np.array_equal(u[0].astype(np.int64), (u0[0].astype(np.int64) + 25 * step) % o.period)
    assert np.array_equal(v1, v)
    assert obs["KEt"][0] == pytest.approx(0.5 * (v[0] @ v[0]), rel=1e-15)


def test_free_rotor_about_principal_axis(oracle_mod):
    """Torque-free rotation about a principal axis: j constant exactly,
    |q| = 1, angle = omega t (SPEC S:317-318 free rotor)."""
    comp = S.c3_component()
    Iz = comp["inertia"][2]
    omega = 0.01 / 0.5
    s, c, r, v, q, j = lone(comp, box=200.0, rc=18.9, j=(0, 0, Iz * omega))
    o = oracle_mod.System(s)
    dt, n = 0.005, 400                              # omega dt = 1e-3
    u, _, q1, j1, obs = o.run(dt, c, o.quantize(r), v, q, j, n, half_step=1, mode="brute")
    assert np.array_equal(j1, j)
    assert abs(np.linalg.norm(q1[0]) - 1) < 1e-14
    ang = 2 * math.atan2(q1[0, 3], q1[0, 0])
    assert ang == pytest.approx(omega * dt * n, rel=1e-4)
    assert abs(q1[0, 1]) < 1e-14 and abs(q1[0, 2]) < 1e-14
    assert obs["KEr"][0] == pytest.approx(0.5 * Iz * omega ** 2, rel=1e-12)


def rk4_top(I, q, jw, t, h):
    """Independent reference: torque-free rigid body, RK4 on
    dq/dt = 1/2 q (x) (0, w_b), w_b = I^-1 R(q)^T j_world (j_world const)."""
    def R(q):
        w, x, y, z = q
        return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                         [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                         [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])

    def f(q):
        qn = q / np.linalg.norm(q)
        wb = (R(qn).T @ jw) / I
        w, x, y, z = q
        a, b, c = wb
        return 0.5 * np.array([-x * a - y * b - z * c, w * a + y * c - z * b,
                               w * b - x * c + z * a, w * c + x * b - y * a])
    q = np.array(q, float)
    for _ in range(int(round(t / h))):
        k1 = f(q); k2 = f(q + h / 2 * k1); k3 = f(q + h / 2 * k2); k4 = f(q + h * k3)
        q = q + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
    return q / np.linalg.norm(q)


def test_fincham_second_order_asymmetric_top(oracle_mod):
    """Torque-free asymmetric top with config 3's inertia: orientation error
    against an RK4 reference falls ~4x per halving of dt (second order), and
    the rotational kinetic energy spread shrinks ~4x as well."""
    comp = S.c3_component()
    I = np.array(comp["inertia"])
    rng = np.random.default_rng(1)
    jb = rng.normal(size=3) * np.sqrt(I * 1e-3)
    q0 = rng.normal(size=4); q0 /= np.linalg.norm(q0)
    w, x, y, z = q0
    R0 = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                   [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                   [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    jw = R0 @ jb
    T_end = 200 * 0.0306
    ref = rk4_top(I, q0, jw, T_end, 0.0306 / 200)
    errs, spreads = [], []
    for dt in (0.0306, 0.0153, 0.00765):
        n = int(round(T_end / dt))
        s, c, r, v, q, j = lone(comp, box=200.0, rc=18.9, q=tuple(q0), j=tuple(jw))
        o = oracle_mod.System(s)
        _, _, q1, _, obs = o.run(dt, c, o.quantize(r), v, q, j, n, half_step=1, mode="brute")
        qq = q1[0] * np.sign(q1[0] @ ref)
        errs.append(np.linalg.norm(qq - ref))
        spreads.append(np.ptp(obs["KEr"]) / obs["KEr"].mean())
    assert errs[0] / errs[1] > 3.3 and errs[1] / errs[2] > 3.3
    assert spreads[0] / spreads[1] > 3.0 and spreads[1] / spreads[2] > 3.0


def dimer(oracle_mod, dt, n):
    s = {"components": [S.lj1_component()], "box": (20.0,) * 3, "rc": 2.5}
    o = oracle_mod.System(s)
    r = np.array([[10.0, 10, 10], [11.3, 10, 10]])
    v = np.array([[0.2, 0, 0], [-0.2, 0, 0]])
    u, v1, _, _, obs = o.run(dt, np.zeros(2, np.int32), o.quantize(r), v,
                             np.tile([1.0, 0, 0, 0], (2, 1)), np.zeros((2, 3)), n,
                             half_step=0, mode="brute")
    return (u[1, 0].astype(np.int64) - u[0, 0].astype(np.int64)) * o.quantum


def test_leapfrog_second_order(oracle_mod):
    """LJ dimer vibration: separation error against a fine-step reference
    falls ~4x per halving of dt (ratio >= 3.8 for a harmonic
    oscillator; the LJ dimer is anharmonic, bound 3.5)."""
    T_end = 2.0
    ref = dimer(oracle_mod, 1e-4, int(T_end / 1e-4))
    e = [abs(dimer(oracle_mod, dt, int(round(T_end / dt))) - ref) for dt in (0.02, 0.01, 0.005)]
    assert e[0] / e[1] > 3.5 and e[1] / e[2] > 3.5


def test_reversibility_translation(oracle_mod):
    """Forward n steps, reverse the on-step velocities, n steps back: the
    fixed-point positions return exactly."""
    s = S.config("c1s")
    o = oracle_mod.System(s)
    u0 = o.quantize(s["r"])
    n, dt = 20, s["dt"]
    u1, vh, q1, j1, _ = o.run(dt, s["comp"], u0, s["v"], s["q"], s["j"], n, 0, "full")
    F, _, _ = o.forces(s["comp"], u1, q1, mode="full")
    v_on = vh + 0.5 * dt * F                        # v(t_n), m = 1
    u2, vh2, _, _, _ = o.run(dt, s["comp"], u1, -v_on, q1, j1, n, 0, "full")
    assert np.array_equal(u2, u0)
    F0, _, _ = o.forces(s["comp"], u2, q1, mode="full")
    assert np.abs(-(vh2 + 0.5 * dt * F0) - s["v"]).max() < 1e-10


def test_initial_temperature_and_nve(oracle_mod):
    """A8: the on-step input velocities give T(0) = generator T exactly;
    NVE over 400 steps of config 0 (lattice melting) keeps
    |E(t) - E(0)| / N <= 2.5e-4 eps; momentum is conserved."""
    s = S.config0()
    o = oracle_mod.System(s)
    u, vh, q, j, obs = o.run(s["dt"], s["comp"], o.quantize(s["r"]), s["v"], s["q"], s["j"],
                             400, 0, "full")
    N = len(u)
    assert obs["T"][0] == pytest.approx(s["T"], rel=1e-12)
    E = obs["U"] + obs["KEt"] + obs["KEr"]
    assert np.abs(E - E[0]).max() / N < 2.5e-4
    assert np.abs(E[:10] - E[0]).max() / N < 1e-5
    assert np.abs(vh.sum(0)).max() < 1e-9
    assert (obs["npairs"] > 0).all()
