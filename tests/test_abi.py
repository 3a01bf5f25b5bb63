"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/mardyn.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "mardyn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mardyn_[a-z_]+)\s*\(", src)))


def test_header_matches_binding():
    from paper_1408_4599_b200 import mardyn
    assert declared() == sorted(mardyn.EXPORTS)


def test_library_exports_every_symbol():
    from paper_1408_4599_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    missing = [s for s in declared() if not hasattr(lib, s)]
    assert not missing
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mardyn_\w+)", out))
    assert set(declared()) <= exported


def test_library_is_sm100a():
    from paper_1408_4599_b200 import build
    lib_path = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import scenarios as S
    from paper_1408_4599_b200 import mardyn
    s = S.config0()
    with pytest.raises(RuntimeError):
        mardyn.Context(s["box"], s["rc"], s["components"], s["dt"])


def test_lj_tail_library_equals_oracle(oracle_mod):
    """mardyn_lj_tail (host code of the library) against the oracle's
    independent implementation (itself pinned by quadrature in
    test_oracle_ensembles.py): single component and a mixture with eta."""
    import numpy as np
    import scenarios as S
    from paper_1408_4599_b200 import mardyn
    s = S.config0()
    o = oracle_mod.System(s)
    V = float(np.prod(o.box))
    U, W = mardyn.lj_tail(s["components"], [4000], V, s["rc"])
    Uo, Wo = o.lj_tail([4000], V)
    assert U == pytest.approx(Uo, rel=1e-13) and W == pytest.approx(Wo, rel=1e-13)
    comps = [S.c2_component(), S.lj1_component(sigma=1.2, eps=0.8)]
    eta = np.array([[1.0, 0.9], [0.9, 1.0]])
    s["components"] = comps
    o = oracle_mod.System(s, eta=eta)
    U, W = mardyn.lj_tail(comps, [300, 500], 2000.0, s["rc"], eta=eta)
    Uo, Wo = o.lj_tail([300, 500], 2000.0)
    assert U == pytest.approx(Uo, rel=1e-13) and W == pytest.approx(Wo, rel=1e-13)
