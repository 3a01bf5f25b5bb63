"""Shared helpers of the GPU parity tests: run the CUDA path (through the
C ABI binding) and the fp64 oracle on the same seeded inputs and compare
with the tolerances BASELINE.json's north_star states (reading A15):

  cells / per-cell counts      bit-exact
  forces, torques              max |dF| <= 1e-4 * RMS |F|   (per component)
  U_pot, virial                relative <= 1e-5
  positions after config 0     <= 1e-4 sigma (minimum image)
"""
import numpy as np

F_TOL = 1e-4
E_TOL = 1e-5


def rms(F):
    return float(np.sqrt(np.mean(np.sum(F * F, axis=1))))


def assert_forces_close(Fg, Fo, what="force", tol=F_TOL):
    scale = rms(Fo)
    err = float(np.abs(Fg - Fo).max())
    assert err <= tol * scale, f"{what}: max |d| = {err:.3e} > {tol} * RMS {scale:.3e}"
    return err / scale if scale > 0 else 0.0


def assert_rel(a, b, what, tol=E_TOL):
    rel = abs(a - b) / max(abs(b), 1e-300)
    assert rel <= tol, f"{what}: gpu {a!r} oracle {b!r} rel {rel:.3e} > {tol}"
    return rel


def min_image(d, box):
    return d - box * np.round(d / box)


def candidates_from_counts(count, ncell):
    """Full-shell candidate count sum_c n_c (sum_27 n_j) - N from per-cell counts."""
    nx, ny, nz = ncell
    c = count.reshape(nz, ny, nx).astype(np.int64)
    nb = sum(np.roll(c, (dz, dy, dx), axis=(0, 1, 2))
             for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1))
    return int((c * nb).sum() - c.sum())
