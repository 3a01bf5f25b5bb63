"""The seeded generators reproduce the BASELINE.json state points
 and Table 1's unit algebra."""
import math

import numpy as np
import pytest

import scenarios as S


def test_table1_units():
    """P:99-114 with reading A16: T0 = E0/k_B, t0 = l0 sqrt(m0/E0),
    v0 = l0/t0 (k_B = 1.380649e-23 J/K, m0 = 1 kg/mol per molecule)."""
    kB = 1.380649e-23
    m0 = 1.0 / S.AVOGADRO
    assert S.E0_J / kB == pytest.approx(S.T0_K, rel=2e-6)
    assert S.BOHR_M * math.sqrt(m0 / S.E0_J) == pytest.approx(S.T0_S, rel=2e-6)
    assert S.BOHR_M / S.T0_S == pytest.approx(1620.35, rel=2e-5)   # printed to 6 digits


@pytest.mark.parametrize("name,N,rho,T", [("c0", 4000, 0.6, 0.7), ("c1s", 4000, 0.75, 0.95)])
def test_lj_configs(name, N, rho, T):
    s = S.config(name)
    assert len(s["r"]) == N
    assert N / np.prod(s["box"]) == pytest.approx(rho, rel=1e-12)
    assert np.sum(s["v"] ** 2) / (3 * N) == pytest.approx(T, rel=1e-12)
    assert np.abs(s["v"].sum(0)).max() < 1e-9
    assert (s["r"] >= 0).all() and (s["r"] < s["box"]).all()


def test_rigid_configs():
    s = S.config("c2s")
    assert len(s["r"]) == 16 ** 3 and s["rc"] == 4.0 and s["dt"] == 0.001
    assert np.allclose(np.linalg.norm(s["q"], axis=1), 1)
    s = S.config("c3s")
    c = s["components"][0]
    assert c["mass"] == pytest.approx(0.0180154, rel=1e-6)
    assert s["T"] == pytest.approx(298 / 315775)
    assert s["rc"] == pytest.approx(18.8973, rel=1e-5)


def test_slab_config():
    s = S.config("c4s")
    z = s["r"][:, 2]
    Lz = s["box"][2]
    mid = (z > Lz / 3 + 2) & (z < 2 * Lz / 3 - 2)
    rho_l = mid.sum() / (s["box"][0] * s["box"][1] * (Lz / 3 - 4))
    assert rho_l == pytest.approx(0.724, rel=0.02)
    vap = (z < Lz / 3 - 3) | (z > 2 * Lz / 3 + 3)
    rho_v = vap.sum() / (s["box"][0] * s["box"][1] * (2 * Lz / 3 - 6 - 2 * 0.0))
    assert 0.01 < rho_v < 0.03
