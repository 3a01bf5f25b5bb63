"""Pins of the oracle's NEXT-row additions (not GPU):
isotropic LJ tail corrections (reading A3: reported beside
U_pot, not in it) against numerical quadrature of the mean-field integral,
and NVT velocity rescaling (reading A24) against hand values."""
import math

import numpy as np
import pytest
from scipy import integrate

import scenarios as S


def u_lj(r, sig, eps):
    return 4 * eps * ((sig / r) ** 12 - (sig / r) ** 6)


def du_lj(r, sig, eps):
    return 4 * eps * (-12 * sig ** 12 / r ** 13 + 6 * sig ** 6 / r ** 7)


def quad_tail(sig, eps, rc):
    """int_rc^inf u 4 pi r^2 dr and int_rc^inf r u' 4 pi r^2 dr by quadrature."""
    iu = integrate.quad(lambda r: u_lj(r, sig, eps) * 4 * math.pi * r * r, rc, np.inf, epsabs=0, epsrel=1e-12)[0]
    iw = integrate.quad(lambda r: r * du_lj(r, sig, eps) * 4 * math.pi * r * r, rc, np.inf, epsabs=0,
                        epsrel=1e-12)[0]
    return iu, iw


@pytest.mark.parametrize("rho,rc", [(0.6223, 2.5), (0.75, 2.5), (0.3, 4.0)])
def test_lj_tail_matches_quadrature(oracle_mod, rho, rc):
    """U_lrc/N = rho/2 int u 4 pi r^2 dr (the value for
    rho = 0.6223, rc = 2.5 to 1e-8), W_lrc/N = -rho/2 int r u' 4 pi r^2 dr."""
    s = S.config0()
    s["rc"] = rc
    o = oracle_mod.System(s)
    N = 1000
    V = N / rho
    U, W = o.lj_tail([N], V)
    iu, iw = quad_tail(1.0, 1.0, rc)
    assert U / N == pytest.approx(0.5 * rho * iu, rel=1e-8)
    assert W / N == pytest.approx(-0.5 * rho * iw, rel=1e-8)
    # closed form of the per-molecule energy
    x3 = (1.0 / rc) ** 3
    assert U / N == pytest.approx(8 / 3 * math.pi * rho * (x3 ** 3 / 3 - x3), rel=1e-12)


def test_lj_tail_limits(oracle_mod):
    """rho = 0 -> 0; rc -> 1e3 sigma -> below 1e-8 eps."""
    s = S.config0()
    o = oracle_mod.System(s)
    assert o.lj_tail([0], 1000.0) == (0.0, 0.0)
    s["rc"] = 1.0e3
    s["box"] = (3.5e3,) * 3
    o = oracle_mod.System(s)
    U, W = o.lj_tail([1000], 1000 / 0.8)
    assert abs(U) / 1000 < 1e-8
    assert W / 1000 == pytest.approx(16 / 3 * math.pi * 0.8 * (2e-27 - 3e-9), rel=1e-9)


def test_lj_tail_mixture_and_sites(oracle_mod):
    """Two components (2CLJQ with two LJ sites, single-site LJ with sigma 1.2),
    unlike-pair eta: the sum over ordered component pairs and LJ site
    pairs of N_a N_b / (2V) times the quadrature integrals, Lorentz-Berthelot."""
    c2 = S.c2_component()
    c1 = S.lj1_component(sigma=1.2, eps=0.8)
    s = S.config0()
    s["components"] = [c2, c1]
    eta = np.array([[1.0, 0.9], [0.9, 1.0]])
    o = oracle_mod.System(s, eta=eta)
    counts, V = [300, 500], 2000.0
    U, W = o.lj_tail(counts, V)
    sites = [[(x[1], x[2]) for x in c2["lj"]], [(x[1], x[2]) for x in c1["lj"]]]
    eu = ew = 0.0
    for a in range(2):
        for b in range(2):
            for sa, ea in sites[a]:
                for sb, eb in sites[b]:
                    sig, eps = 0.5 * (sa + sb), eta[a, b] * math.sqrt(ea * eb)
                    iu, iw = quad_tail(sig, eps, s["rc"])
                    eu += 0.5 * counts[a] * counts[b] / V * iu
                    ew -= 0.5 * counts[a] * counts[b] / V * iw
    assert U == pytest.approx(eu, rel=1e-8)
    assert W == pytest.approx(ew, rel=1e-8)


def test_nvt_rescale_hand_values(oracle_mod):
    """lambda = sqrt(T_target / T).  T_target = T(t_0) / 4
    halves every half-step velocity of the NVE step; T_target = T(t_0)
    leaves it unchanged (lambda = 1, up to the rounding of sqrt(x/x))."""
    s = S.config0()
    o = oracle_mod.System(s)
    u0 = o.quantize(s["r"])
    args = (s["dt"], s["comp"], u0, s["v"], s["q"], s["j"], 1)
    _, v_nve, _, _, obs = o.run(*args, half_step=0, mode="full")
    T0 = obs["T"][0]
    _, v_q, _, _, _ = o.run(*args, half_step=0, mode="full", T_target=T0 / 4, thermostat_interval=1)
    assert np.allclose(v_q, 0.5 * v_nve, rtol=1e-14, atol=0)
    _, v_1, _, _, _ = o.run(*args, half_step=0, mode="full", T_target=T0, thermostat_interval=1)
    assert np.allclose(v_1, v_nve, rtol=1e-15, atol=0)


def test_nvt_holds_temperature(oracle_mod):
    """Rescaling every 5 steps toward T = 1.2 from the T = 0.7 lattice: the
    temperatures right after each rescale move to the target and stay closer
    to it than in the NVE run; the cadence is exactly every 5 steps."""
    s = S.config0()
    o = oracle_mod.System(s)
    u0 = o.quantize(s["r"])
    n = 40
    _, _, _, _, nve = o.run(s["dt"], s["comp"], u0, s["v"], s["q"], s["j"], n, mode="full")
    _, _, _, _, nvt = o.run(s["dt"], s["comp"], u0, s["v"], s["q"], s["j"], n, mode="full",
                            T_target=1.2, thermostat_interval=5)
    assert np.array_equal(nve["T"][:5], nvt["T"][:5])           # untouched before the first rescale
    assert abs(nvt["T"][5] - 1.2) < 0.05 < abs(nve["T"][5] - 1.2)
    assert np.abs(nvt["T"][-10:] - 1.2).max() < 0.1
