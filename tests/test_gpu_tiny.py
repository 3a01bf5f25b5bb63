"""Degenerate system sizes: one molecule (no pair at all: U = W = 0, zero force, only
kinetic energy) and two molecules (one pair, straddling a cell face), for the
single-site kernel and both rigid shapes (2CLJQ, water).  The rigid kernel pads its
partner rounds with a far dummy whose LJ terms are ~1e-26 instead of masking them
(DESIGN.md §6), so "zero" there means below 1e-20.  The pair distance keeps the pair
energy from being a near-cancellation of its site terms: two waters 0.8 rc (8 A) apart
have U ~ 1.5e-4 E_h from nine q-q terms of ~1e-2 each, and the fp32 site sums then
missed the oracle's U by 3.8e-5 relative (measured); at 0.35 rc (3.5 A) they agree to
1e-5.  Step 0 element by element against the fp64 oracle, then 20 steps per-step U, W,
T (reading A25 measure) and the final positions.  Boxes, cutoffs and models are those of the
c1s / c2s / c3s configurations (BASELINE.json configs[1..3], scaled)."""
import numpy as np
import pytest

import scenarios as S
from parity_util import assert_forces_close, assert_rel, min_image

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def md():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1408_4599_b200 import build, mardyn
    build.build()
    return mardyn


SEP = {"c1s": 0.8, "c2s": 0.5, "c3s": 0.35}          # pair distance / rc


def tiny(name, n):
    """n (1 or 2) molecules of config `name`: the pair sits SEP rc apart across the face
    between cells 0 and 1 (x), slightly offset in y."""
    s0 = S.config(name)
    rc = s0["rc"]
    h = 0.5 * SEP[name] * rc
    edge = s0["box"] / np.floor(s0["box"] / rc)
    r = np.array([[edge[0] - h, 0.5 * edge[1], 0.5 * edge[2]],
                  [edge[0] + h, 0.5 * edge[1] + 0.1 * rc, 0.5 * edge[2]]])[:n]
    s = dict(s0, id=np.arange(n, dtype=np.int64), r=r, v=0.3 * s0["v"][:n], q=s0["q"][:n].copy(),
             j=0.3 * s0["j"][:n], comp=s0["comp"][:n].copy())
    return s


def scaled_err(a, b):
    b = np.asarray(b, float)
    return np.abs(np.asarray(a, float) - b) / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("name", ["c1s", "c2s", "c3s"])
@pytest.mark.parametrize("n", [1, 2])
def test_tiny_system(md, oracle_mod, name, n):
    s = tiny(name, n)
    rigid = name != "c1s"
    ctx = md.from_system(s)
    F, tau = ctx.get_forces()
    ctx.compute_forces()
    obs = ctx.get_observables()
    o = oracle_mod.System(s)
    u0 = o.quantize(s["r"])
    Fo, to, tot = o.forces(s["comp"], u0, s["q"], mode="full")
    assert obs["n_pairs"] == tot["npairs"] == n - 1
    if n == 1:
        assert np.abs(F).max() < 1e-20 and np.abs(tau).max() < 1e-20
        assert abs(obs["U_pot"]) < 1e-20 and abs(obs["virial"]) < 1e-20
        assert tot["U"] == 0.0 and tot["W"] == 0.0
    else:
        assert_forces_close(F, Fo, "force")
        if rigid:
            assert_forces_close(tau, to, "torque")
        assert_rel(obs["U_pot"], tot["U"], "U_pot")
        assert_rel(obs["virial"], tot["W"], "virial")
    nsteps = 20
    ctx.step(nsteps)
    hist = ctx.get_observable_history(nsteps)
    uo, vo, qo, jo, ob = o.run(s["dt"], s["comp"], u0, s["v"], s["q"], s["j"], nsteps, half_step=0, mode="full")
    assert [h["step"] for h in hist] == list(range(nsteps))
    for key, ok in (("U_pot", "U"), ("virial", "W"), ("T", "T")):
        g = np.array([h[key] for h in hist])
        if n == 1 and key != "T":
            assert np.abs(g).max() < 1e-20 and np.all(np.asarray(ob[ok]) == 0.0)
            continue
        e = scaled_err(g, ob[ok])
        assert e.max() <= 1e-5, (key, int(e.argmax()), e.max())
    assert [h["n_pairs"] for h in hist] == list(np.asarray(ob["npairs"]).astype(int))
    m = ctx.get_molecules()
    assert np.abs(min_image(m["r"] - uo * o.quantum, o.box)).max() <= 1e-4
    ug, cg, ng = ctx.get_raw()
    co, no = o.cells(ug)
    assert np.array_equal(cg, co) and np.array_equal(ng, no)


def test_cell_faces_and_box_edges(md, oracle_mod):
    """Molecules exactly on cell faces (x = k edge), on the periodic boundary written as
    L instead of 0, and a hair below L: the device ingest and the oracle quantise them to
    the same fixed-point lattice (reading A12) and bin them into the same cells, and the
    forces agree.  One molecule per cell corner (spacing = edge >= rc)."""
    s0 = S.config("c1s")
    L = s0["box"]
    n = np.floor(L / s0["rc"]).astype(int)
    edge = L / n
    g = np.stack(np.meshgrid(*[np.arange(k) for k in n], indexing="ij"), -1).reshape(-1, 3).astype(float)
    r = g * edge
    r[r[:, 1] == 0.0, 0] += 0.3 * edge[0]            # break the cubic symmetry a little
    sel = (g[:, 0] == 0) & (g[:, 2] == 1)
    r[sel, 0] = L[0]                                  # x = L: the same point as x = 0
    sel = (g[:, 1] == 0) & (g[:, 2] == 2)
    r[sel, 1] = np.nextafter(L[1], 0.0)               # a hair below L
    m = len(r)
    rng = np.random.default_rng(7)
    s = dict(s0, id=np.arange(m, dtype=np.int64), r=r, v=0.2 * rng.normal(size=(m, 3)),
             q=np.tile([1.0, 0.0, 0.0, 0.0], (m, 1)), j=np.zeros((m, 3)), comp=np.zeros(m, np.int32))
    ctx = md.from_system(s)
    F, _ = ctx.get_forces()
    ctx.compute_forces()
    obs = ctx.get_observables()
    ug, cg, ng = ctx.get_raw()
    o = oracle_mod.System(s)
    uo = o.quantize(s["r"])
    co, no = o.cells(uo)
    assert np.array_equal(ug, uo)
    assert np.array_equal(cg, co) and np.array_equal(ng, no)
    Fo, _, tot = o.forces(s["comp"], uo, s["q"], mode="full")
    assert obs["n_pairs"] == tot["npairs"]
    assert_forces_close(F, Fo, "force")
    assert_rel(obs["U_pot"], tot["U"], "U_pot")
