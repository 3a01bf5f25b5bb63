"""ctypes wrapper of the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  It shares no code with the CUDA path (``paper_1408_4599_b200``)
and never imports it; its inputs come from ``scenarios`` (seeded generators)
only.  See the header of oracle.c for what is computed and the paper passages
each function follows.

Parity pins: every function here is pinned in tests/test_oracle_*.py against
closed forms, brute force, point-charge limits, finite differences and
conservation laws.  Reading A17 (the TIP4P constants of
config 3) has no published reference for this exact variant in the container:
the *physical realism* of config 3 is "parity unpinned"; its arithmetic is
pinned by the generic site-pair pins.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_LJ, OR_CHARGE, OR_DIPOLE, OR_QUADRUPOLE = 0, 1, 2, 3


def build(force=False):
    """Compile oracle.c with gcc (plain C, OpenMP for the full-shell leg)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-std=c11", "-Wall", "-shared",
                               "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class Site(C.Structure):
    _fields_ = [("type", C.c_int32), ("pad", C.c_int32), ("r", C.c_double * 3),
                ("e", C.c_double * 3), ("m", C.c_double), ("sigma", C.c_double),
                ("eps", C.c_double)]


class Comp(C.Structure):
    _fields_ = [("mass", C.c_double), ("I", C.c_double * 3), ("site0", C.c_int32),
                ("nsites", C.c_int32)]


class Sys(C.Structure):
    _fields_ = [("L", C.c_double * 3), ("rc", C.c_double), ("eps_rf", C.c_double),
                ("lj_shift", C.c_int32), ("n_comp", C.c_int32),
                ("comp", C.POINTER(Comp)), ("sites", C.POINTER(Site)),
                ("eta", C.POINTER(C.c_double)),
                ("nc", C.c_int32 * 3), ("E", C.c_int64 * 3), ("P", C.c_int64 * 3),
                ("s", C.c_double), ("box", C.c_double * 3)]


class Totals(C.Structure):
    _fields_ = [("U", C.c_double), ("W", C.c_double), ("npairs", C.c_int64)]


class Obs(C.Structure):
    _fields_ = [("U", C.c_double), ("W", C.c_double), ("KEt", C.c_double),
                ("KEr", C.c_double), ("T", C.c_double), ("npairs", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        _lib.or_setup.argtypes = [P(Sys)]
        _lib.or_quantize.argtypes = [P(Sys), C.c_int64, C.c_void_p, C.c_void_p]
        _lib.or_cells.argtypes = [P(Sys), C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.or_site_pair.argtypes = [P(Sys), P(Site), C.c_void_p, P(Site), C.c_void_p,
                                      C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]
        fargs = [P(Sys), C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                 C.c_void_p, P(Totals)]
        _lib.or_forces_brute.argtypes = fargs
        _lib.or_forces_cells.argtypes = fargs
        _lib.or_forces_full.argtypes = [P(Sys), C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        _lib.or_run.argtypes = [P(Sys), C.c_double, C.c_int64, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                C.c_int, C.c_int, P(Obs)]
        _lib.or_run_nvt.argtypes = [P(Sys), C.c_double, C.c_int64, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_double, C.c_int, P(Obs)]
        _lib.or_run_cont.argtypes = [P(Sys), C.c_double, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, P(Obs)]
        _lib.or_lj_tail.argtypes = [P(Sys), C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def make_site(kind, pos, axis=(0, 0, 0), m=0.0, sigma=0.0, eps=0.0):
    s = Site()
    s.type = kind
    s.r[:] = list(map(float, pos))
    s.e[:] = list(map(float, axis))
    s.m, s.sigma, s.eps = float(m), float(sigma), float(eps)
    return s


class System:
    """Oracle view of a scenarios system dict (components, box, cutoff)."""

    def __init__(self, system, L=None, rc=None, eta=None):
        comps = system["components"]
        sites, cs = [], []
        for cd in comps:
            c = Comp()
            c.mass = cd["mass"]
            c.I[:] = list(cd["inertia"])
            c.site0 = len(sites)
            for p, sg, ep in cd["lj"]:
                sites.append(make_site(OR_LJ, p, sigma=sg, eps=ep))
            for p, q in cd["charges"]:
                sites.append(make_site(OR_CHARGE, p, m=q))
            for p, a, m in cd["dipoles"]:
                sites.append(make_site(OR_DIPOLE, p, a, m))
            for p, a, m in cd["quadrupoles"]:
                sites.append(make_site(OR_QUADRUPOLE, p, a, m))
            c.nsites = len(sites) - c.site0
            cs.append(c)
        self._sites = (Site * max(len(sites), 1))(*sites)
        self._comps = (Comp * len(cs))(*cs)
        self.s = Sys()
        self.s.L[:] = list(map(float, system["box"] if L is None else L))
        self.s.rc = float(system["rc"] if rc is None else rc)
        self.s.eps_rf = float(system.get("eps_rf", math.inf))
        self.s.lj_shift = int(system.get("lj_shift", 1))
        self.s.n_comp = len(cs)
        self.s.comp = C.cast(self._comps, C.POINTER(Comp))
        self.s.sites = C.cast(self._sites, C.POINTER(Site))
        self._eta = None
        if eta is not None:
            self._eta = np.ascontiguousarray(eta, dtype=np.float64)
            self.s.eta = self._eta.ctypes.data_as(C.POINTER(C.c_double))
        if lib().or_setup(C.byref(self.s)) != 0:
            raise ValueError("oracle: invalid box / cutoff")

    # grid (reading A12)
    @property
    def ncell(self):
        return tuple(self.s.nc)

    @property
    def quantum(self):
        return self.s.s

    @property
    def box(self):
        return np.array(self.s.box[:])

    @property
    def period(self):
        return np.array(self.s.P[:], dtype=np.int64)

    @property
    def edge_q(self):
        return np.array(self.s.E[:], dtype=np.int64)

    def quantize(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        u = np.empty(r.shape, dtype=np.uint32)
        lib().or_quantize(C.byref(self.s), len(r), _ptr(r), _ptr(u))
        return u

    def cells(self, u):
        u = np.ascontiguousarray(u, dtype=np.uint32)
        n = len(u)
        cell = np.empty(n, np.int32)
        count = np.empty(int(np.prod(self.ncell)), np.int32)
        lib().or_cells(C.byref(self.s), n, _ptr(u), _ptr(cell), _ptr(count))
        return cell, count

    def forces(self, comp, u, q, mode="cells", idx=None, nthreads=0):
        """F, tau per molecule and totals.  mode: 'brute' | 'cells' | 'full'.
        For 'full', idx selects the molecules whose F, tau are returned and the
        totals (U, W, npairs) are those of the selected molecules' halves."""
        comp = np.ascontiguousarray(comp, np.int32)
        u = np.ascontiguousarray(u, np.uint32)
        q = np.ascontiguousarray(q, np.float64)
        n = len(u)
        if mode == "full":
            sel = None if idx is None else np.ascontiguousarray(idx, np.int64)
            m = n if sel is None else len(sel)
            F = np.empty((m, 3)); tau = np.empty((m, 3))
            ui = np.empty(m); wi = np.empty(m); npi = np.empty(m, np.int64)
            rc = lib().or_forces_full(C.byref(self.s), n, _ptr(comp), _ptr(u), _ptr(q), m,
                                      None if sel is None else _ptr(sel), _ptr(F), _ptr(tau),
                                      _ptr(ui), _ptr(wi), _ptr(npi), int(nthreads))
            if rc:
                raise RuntimeError(f"or_forces_full failed ({rc})")
            return F, tau, {"U": float(ui.sum()), "W": float(wi.sum()),
                            "npairs": int(npi.sum()) // (2 if sel is None else 1),
                            "u_i": ui, "w_i": wi, "np_i": npi}
        F = np.empty((n, 3)); tau = np.empty((n, 3))
        tot = Totals()
        fn = lib().or_forces_brute if mode == "brute" else lib().or_forces_cells
        rc = fn(C.byref(self.s), n, _ptr(comp), _ptr(u), _ptr(q), _ptr(F), _ptr(tau),
                C.byref(tot))
        if rc:
            raise RuntimeError(f"oracle forces failed ({rc})")
        return F, tau, {"U": tot.U, "W": tot.W, "npairs": tot.npairs}

    def lj_tail(self, counts, volume):
        """Isotropic LJ tail corrections (U_lrc, W_lrc) for molecule counts per
        component in the given volume (reading A3)."""
        c = np.ascontiguousarray(counts, np.int64)
        U = np.zeros(1); W = np.zeros(1)
        lib().or_lj_tail(C.byref(self.s), _ptr(c), float(volume), _ptr(U), _ptr(W))
        return float(U[0]), float(W[0])

    def run(self, dt, comp, u, v, q, j, nsteps, half_step=0, mode="full", nthreads=0, T_target=0.0,
            thermostat_interval=0):
        """Leapfrog + Fincham for nsteps; returns (u, v, q, j, obs) with obs a
        structured array of per-step (U, W, KEt, KEr, T, npairs) at t_k.
        T_target > 0: NVT velocity rescaling every thermostat_interval steps (A24)."""
        comp = np.ascontiguousarray(comp, np.int32)
        u = np.array(u, dtype=np.uint32, order="C")
        v = np.array(v, dtype=np.float64, order="C")
        q = np.array(q, dtype=np.float64, order="C")
        j = np.array(j, dtype=np.float64, order="C")
        obs = (Obs * max(nsteps, 1))()
        m = {"brute": 0, "cells": 1, "full": 2}[mode]
        rc = lib().or_run_nvt(C.byref(self.s), float(dt), len(u), _ptr(comp), _ptr(u), _ptr(v),
                              _ptr(q), _ptr(j), int(nsteps), int(half_step), m, int(nthreads),
                              float(T_target), int(thermostat_interval), obs)
        if rc:
            raise RuntimeError(f"or_run failed ({rc})")
        out = np.array([(o.U, o.W, o.KEt, o.KEr, o.T, o.npairs) for o in obs[:nsteps]],
                       dtype=[("U", "f8"), ("W", "f8"), ("KEt", "f8"), ("KEr", "f8"),
                              ("T", "f8"), ("npairs", "i8")])
        return u, v, q, j, out

    def run_continuous(self, dt, comp, r, v, q, j, nsteps, half_step=0, nthreads=0):
        """The same steps on unquantised fp64 positions (no A12 lattice; brute-force
        full shell, fp64 minimum image): the reference that bounds the effect of the
        position quantum.  Returns (r, v, q, j, obs) like run()."""
        comp = np.ascontiguousarray(comp, np.int32)
        r = np.array(r, dtype=np.float64, order="C") % self.box
        v = np.array(v, dtype=np.float64, order="C")
        q = np.array(q, dtype=np.float64, order="C")
        j = np.array(j, dtype=np.float64, order="C")
        obs = (Obs * max(nsteps, 1))()
        rc = lib().or_run_cont(C.byref(self.s), float(dt), len(r), _ptr(comp), _ptr(r), _ptr(v), _ptr(q),
                               _ptr(j), int(nsteps), int(half_step), int(nthreads), obs)
        if rc:
            raise RuntimeError(f"or_run_cont failed ({rc})")
        out = np.array([(o.U, o.W, o.KEt, o.KEr, o.T, o.npairs) for o in obs[:nsteps]],
                       dtype=[("U", "f8"), ("W", "f8"), ("KEt", "f8"), ("KEr", "f8"),
                              ("T", "f8"), ("npairs", "i8")])
        return r, v, q, j, out

    def site_pair(self, a, ea, b, eb, rv, eta=1.0):
        """One site pair (Site structs, world axes, rv = x_b - x_a):
        returns u, f_b, tau_a, tau_b."""
        U = np.zeros(1); fb = np.zeros(3); ta = np.zeros(3); tb = np.zeros(3)
        ea = np.ascontiguousarray(ea, np.float64); eb = np.ascontiguousarray(eb, np.float64)
        rv = np.ascontiguousarray(rv, np.float64)
        lib().or_site_pair(C.byref(self.s), C.byref(a), _ptr(ea), C.byref(b), _ptr(eb),
                           float(eta), _ptr(rv), _ptr(U), _ptr(fb), _ptr(ta), _ptr(tb))
        return float(U[0]), fb, ta, tb

    def unquantize(self, u):
        return np.asarray(u, dtype=np.float64) * self.quantum


def system_positions_fp(sys_o, system):
    """Quantised initial positions of a scenarios system in the oracle lattice."""
    return sys_o.quantize(system["r"])
