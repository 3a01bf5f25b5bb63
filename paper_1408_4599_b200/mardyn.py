"""Thin ctypes binding of libmardyn.so (include/mardyn.h), same names as the
C ABI.  Argument marshalling only: every step of the hot path runs in the
CUDA kernels of the library.  PyTorch provides the three pieces of plumbing
the library does not own: the device workspace (a uint8 tensor), the CUDA
stream, and (for multi-process runs) torch.distributed.

There is no CPU fallback: if the shared library is missing or CUDA is
unavailable, constructing a context raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MARDYN_LIB") or os.path.join(_HERE, "libmardyn.so")

MARDYN_OK = 0
ERRORS = {-1: "EINVAL", -2: "EOVERLAP", -3: "EUNSTABLE", -4: "ECAPACITY", -5: "ECUDA",
          -6: "ENCCL", -7: "ESTATE"}

# every symbol declared in include/mardyn.h
EXPORTS = ["mardyn_create", "mardyn_get_grid", "mardyn_workspace_bytes", "mardyn_set_workspace",
           "mardyn_set_molecules", "mardyn_compute_forces", "mardyn_step", "mardyn_get_observables",
           "mardyn_get_observable_history", "mardyn_get_molecules", "mardyn_get_forces",
           "mardyn_get_raw", "mardyn_last_step_timing", "mardyn_set_profiling",
           "mardyn_launch_count", "mardyn_cell_cost", "mardyn_kd_decompose",
           "mardyn_nccl_unique_id", "mardyn_create_distributed", "mardyn_create_loopback",
           "mardyn_partition", "mardyn_set_partition", "mardyn_get_partition", "mardyn_dd_counts",
           "mardyn_rebalance", "mardyn_grid_counts", "mardyn_kd_partition", "mardyn_set_cost_model",
           "mardyn_set_thermostat", "mardyn_lj_tail", "mardyn_get_tail_corrections",
           "mardyn_last_error", "mardyn_destroy"]


class MardynError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"mardyn {ERRORS.get(code, code)}: {msg}")
        self.code = code


class LJSite(C.Structure):
    _fields_ = [("r", C.c_double * 3), ("sigma", C.c_double), ("epsilon", C.c_double)]


class Charge(C.Structure):
    _fields_ = [("r", C.c_double * 3), ("q", C.c_double)]


class Polar(C.Structure):
    _fields_ = [("r", C.c_double * 3), ("e", C.c_double * 3), ("m", C.c_double)]


class Component(C.Structure):
    _fields_ = [("n_lj", C.c_int32), ("n_q", C.c_int32), ("n_mu", C.c_int32), ("n_Q", C.c_int32),
                ("lj", C.POINTER(LJSite)), ("q", C.POINTER(Charge)), ("mu", C.POINTER(Polar)),
                ("Q", C.POINTER(Polar)), ("mass", C.c_double), ("inertia", C.c_double * 3)]


class Options(C.Structure):
    _fields_ = [("dt", C.c_double), ("eps_rf", C.c_double), ("lj_shift", C.c_int32),
                ("eta", C.POINTER(C.c_double)), ("rebalance_interval", C.c_int32),
                ("cuda_stream", C.c_void_p)]


class Observables(C.Structure):
    _fields_ = [("step", C.c_int64), ("U_pot", C.c_double), ("virial", C.c_double), ("T", C.c_double),
                ("E_kin_trans", C.c_double), ("E_kin_rot", C.c_double), ("n_pairs", C.c_int64),
                ("n_candidates", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Grid(C.Structure):
    _fields_ = [("ncell", C.c_int32 * 3), ("pad", C.c_int32), ("quantum", C.c_double),
                ("period", C.c_int64 * 3), ("edge", C.c_int64 * 3), ("box", C.c_double * 3),
                ("cut2_q", C.c_int64), ("kernel", C.c_int32), ("n_slots", C.c_int32)]


_lib = None


def load_library():
    """Load the in-tree sm_100a library; fails loudly if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1408_4599_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    lib.mardyn_create.argtypes = [P(C.c_double), C.c_double, P(Component), C.c_int32, P(Options), P(vp)]
    lib.mardyn_get_grid.argtypes = [vp, P(Grid)]
    lib.mardyn_workspace_bytes.argtypes = [vp, C.c_int64, P(C.c_size_t)]
    lib.mardyn_set_workspace.argtypes = [vp, vp, C.c_size_t, C.c_int64]
    lib.mardyn_set_molecules.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp, vp, C.c_int32]
    lib.mardyn_compute_forces.argtypes = [vp]
    lib.mardyn_step.argtypes = [vp, C.c_int32]
    lib.mardyn_get_observables.argtypes = [vp, P(Observables)]
    lib.mardyn_get_observable_history.argtypes = [vp, C.c_int32, P(C.c_int32), P(Observables)]
    lib.mardyn_get_molecules.argtypes = [vp, C.c_int64, P(C.c_int64), vp, vp, vp, vp, vp, vp]
    lib.mardyn_get_forces.argtypes = [vp, C.c_int64, vp, vp, P(C.c_int64), vp]
    lib.mardyn_nccl_unique_id.argtypes = [vp]
    lib.mardyn_create_distributed.argtypes = [P(C.c_double), C.c_double, P(Component), C.c_int32, P(Options), vp,
                                              C.c_int32, C.c_int32, C.c_int32, P(vp)]
    lib.mardyn_create_loopback.argtypes = [P(C.c_double), C.c_double, P(Component), C.c_int32, P(Options),
                                           C.c_int32, P(vp)]
    lib.mardyn_partition.argtypes = [vp, C.c_int64, vp]
    lib.mardyn_set_partition.argtypes = [vp, vp]
    lib.mardyn_get_partition.argtypes = [vp, vp]
    lib.mardyn_dd_counts.argtypes = [vp, C.c_int64, vp, vp]
    lib.mardyn_rebalance.argtypes = [vp]
    lib.mardyn_set_cost_model.argtypes = [vp, C.c_int32]
    lib.mardyn_grid_counts.argtypes = [P(C.c_double), C.c_double, C.c_int64, vp, vp, vp]
    lib.mardyn_kd_partition.argtypes = [P(C.c_double), C.c_double, C.c_int64, vp, C.c_int32, vp, vp]
    lib.mardyn_set_thermostat.argtypes = [vp, C.c_double, C.c_int32]
    lib.mardyn_lj_tail.argtypes = [P(Component), C.c_int32, vp, vp, C.c_double, C.c_double, P(C.c_double),
                                   P(C.c_double)]
    lib.mardyn_get_tail_corrections.argtypes = [vp, P(C.c_double), P(C.c_double)]
    lib.mardyn_get_raw.argtypes = [vp, C.c_int64, vp, vp, vp]
    lib.mardyn_last_step_timing.argtypes = [vp, P(C.c_double), P(C.c_double), P(C.c_int32)]
    lib.mardyn_set_profiling.argtypes = [vp, C.c_int32]
    lib.mardyn_launch_count.argtypes = [vp]
    lib.mardyn_launch_count.restype = C.c_int64
    lib.mardyn_cell_cost.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, vp]
    lib.mardyn_kd_decompose.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp, vp]
    lib.mardyn_last_error.argtypes = [vp]
    lib.mardyn_last_error.restype = C.c_char_p
    lib.mardyn_destroy.argtypes = [vp]
    lib.mardyn_destroy.restype = None
    _lib = lib
    return lib


def _host_ptr(a, dtype):
    """Pointer to a C-contiguous host buffer (numpy array or CPU torch tensor,
    pinned or not).  Returns (pointer, keep-alive object)."""
    if a is None:
        return None, None
    try:
        import torch
        if isinstance(a, torch.Tensor):
            assert a.device.type == "cpu" and a.is_contiguous()
            return C.c_void_p(a.data_ptr()), a
    except ImportError:
        pass
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data_as(C.c_void_p), arr


def _out_ptr(a):
    """Writable pointer to a caller-provided C-contiguous host output buffer
    (numpy array or CPU torch tensor, e.g. pinned); never copies."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        assert a.device.type == "cpu" and a.is_contiguous()
        return C.c_void_p(a.data_ptr())
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def _components(components):
    """scenarios-style component dicts -> ctypes array (+ keep-alive list)."""
    keep = []
    arr = (Component * len(components))()
    for c, cd in zip(arr, components):
        lj = (LJSite * max(1, len(cd["lj"])))(*[LJSite((C.c_double * 3)(*p), s, e) for p, s, e in cd["lj"]])
        qq = (Charge * max(1, len(cd["charges"])))(*[Charge((C.c_double * 3)(*p), q) for p, q in cd["charges"]])
        mu = (Polar * max(1, len(cd["dipoles"])))(*[Polar((C.c_double * 3)(*p), (C.c_double * 3)(*a), m)
                                                     for p, a, m in cd["dipoles"]])
        QQ = (Polar * max(1, len(cd["quadrupoles"])))(*[Polar((C.c_double * 3)(*p), (C.c_double * 3)(*a), m)
                                                         for p, a, m in cd["quadrupoles"]])
        keep += [lj, qq, mu, QQ]
        c.n_lj, c.n_q, c.n_mu, c.n_Q = (len(cd["lj"]), len(cd["charges"]), len(cd["dipoles"]),
                                        len(cd["quadrupoles"]))
        c.lj = C.cast(lj, C.POINTER(LJSite)); c.q = C.cast(qq, C.POINTER(Charge))
        c.mu = C.cast(mu, C.POINTER(Polar)); c.Q = C.cast(QQ, C.POINTER(Polar))
        c.mass = cd["mass"]
        c.inertia[:] = list(cd["inertia"])
    return arr, keep


class Context:
    """One simulation box on the current CUDA device (mardyn_ctx)."""

    def __init__(self, box, cutoff, components, dt, eps_rf=math.inf, lj_shift=1, eta=None,
                 capacity=None, stream=None, rebalance_interval=0, _handle=None, _keep=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("mardyn needs a CUDA device (there is no CPU fallback)")
        self.lib = load_library()
        self.torch = torch
        self.stream = stream if stream is not None else torch.cuda.Stream()
        self.ws = None
        self.capacity = 0
        self.rank, self.nranks = 0, 1
        if _handle is not None:                  # a rank of a group made by create_loopback
            self.h, self._keep = _handle, _keep
            return
        self.h = None
        opt, box_a, comps, n = self._options(box, components, dt, eps_rf, lj_shift, eta, rebalance_interval)
        h = C.c_void_p()
        rc = self.lib.mardyn_create(box_a, float(cutoff), comps, n, C.byref(opt), C.byref(h))
        self.h = h
        self._check(rc)
        if capacity is not None:
            self.reserve(capacity)

    def _options(self, box, components, dt, eps_rf, lj_shift, eta, rebalance_interval):
        comps, self._keep = _components(components)
        self._eta = None if eta is None else np.ascontiguousarray(eta, dtype=np.float64)
        opt = Options()
        opt.dt = float(dt)
        opt.eps_rf = float(eps_rf)
        opt.lj_shift = int(lj_shift)
        opt.eta = None if self._eta is None else self._eta.ctypes.data_as(C.POINTER(C.c_double))
        opt.rebalance_interval = int(rebalance_interval)
        opt.cuda_stream = C.c_void_p(self.stream.cuda_stream)
        box_a = (C.c_double * 3)(*[float(x) for x in box])
        return opt, box_a, comps, len(components)

    @classmethod
    def distributed(cls, box, cutoff, components, dt, nccl_id, rank, world, device=None, eps_rf=math.inf,
                    lj_shift=1, eta=None, stream=None, rebalance_interval=0):
        """One rank of a decomposed run over NCCL (mardyn_create_distributed); nccl_id:
        the 128 bytes of rank 0's nccl_unique_id(), broadcast by the caller."""
        import torch
        self = cls.__new__(cls)
        self.lib = load_library()
        self.torch = torch
        dev = torch.cuda.current_device() if device is None else int(device)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=dev)
        self.ws, self.capacity, self.h = None, 0, None
        opt, box_a, comps, n = self._options(box, components, dt, eps_rf, lj_shift, eta, rebalance_interval)
        uid = C.create_string_buffer(bytes(nccl_id), 128)
        h = C.c_void_p()
        rc = self.lib.mardyn_create_distributed(box_a, float(cutoff), comps, n, C.byref(opt), uid, int(rank),
                                                int(world), dev, C.byref(h))
        self.h = h
        self._check(rc)
        self.rank, self.nranks = int(rank), int(world)
        return self

    @classmethod
    def loopback(cls, box, cutoff, components, dt, p, eps_rf=math.inf, lj_shift=1, eta=None, stream=None,
                 rebalance_interval=0):
        """p ranks of a decomposed run in this process on the current device, one
        stream (mardyn_create_loopback): returns their contexts in rank order."""
        import torch
        lead = cls.__new__(cls)
        lead.lib = load_library()
        lead.torch = torch
        lead.stream = stream if stream is not None else torch.cuda.Stream()
        lead.ws, lead.capacity, lead.h = None, 0, None
        opt, box_a, comps, n = lead._options(box, components, dt, eps_rf, lj_shift, eta, rebalance_interval)
        hs = (C.c_void_p * p)()
        rc = lead.lib.mardyn_create_loopback(box_a, float(cutoff), comps, n, C.byref(opt), int(p), hs)
        out = [cls(None, None, None, None, stream=lead.stream, _handle=C.c_void_p(hs[r]), _keep=lead._keep)
               for r in range(p)]
        for r, c in enumerate(out):
            c.rank, c.nranks = r, p
        if rc != MARDYN_OK:
            msg = lead.lib.mardyn_last_error(out[0].h).decode() if hs[0] else ""
            raise MardynError(rc, msg)
        return out

    # -- plumbing ---------------------------------------------------------
    def _check(self, rc):
        if rc != MARDYN_OK:
            msg = self.lib.mardyn_last_error(self.h).decode() if self.h else ""
            raise MardynError(rc, msg)

    def reserve(self, capacity, alloc=None):
        """Allocate the device workspace through PyTorch (caching allocator, or alloc(nbytes),
        e.g. symmetric memory that peers can address)."""
        nbytes = C.c_size_t()
        self._check(self.lib.mardyn_workspace_bytes(self.h, int(capacity), C.byref(nbytes)))
        if alloc is not None:
            self.ws = alloc(nbytes.value + 256)
        else:
            self.ws = self.torch.empty(nbytes.value + 256, dtype=self.torch.uint8, device="cuda")
        ptr = self.ws.data_ptr()
        ptr += (-ptr) % 256
        self._check(self.lib.mardyn_set_workspace(self.h, C.c_void_p(ptr), nbytes.value, int(capacity)))
        self.capacity = int(capacity)

    def close(self):
        if getattr(self, "h", None):
            self.lib.mardyn_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- C ABI, same names -------------------------------------------------
    def get_grid(self):
        g = Grid()
        self._check(self.lib.mardyn_get_grid(self.h, C.byref(g)))
        return {"ncell": tuple(g.ncell), "quantum": g.quantum, "period": tuple(g.period),
                "edge": tuple(g.edge), "box": tuple(g.box), "cut2_q": g.cut2_q,
                "kernel": g.kernel, "n_slots": g.n_slots}

    def set_molecules(self, r, v, comp=None, q=None, j=None, id=None, half_step=0):
        n = len(r)
        if self.capacity < n:
            self.reserve(n)
        if comp is None:
            comp = np.zeros(n, np.int32)
        ptrs = [_host_ptr(x, dt) for x, dt in ((id, np.int64), (comp, np.int32), (r, np.float64),
                                               (v, np.float64), (q, np.float64), (j, np.float64))]
        self._check(self.lib.mardyn_set_molecules(self.h, n, *[p for p, _ in ptrs], int(half_step)))

    def compute_forces(self):
        self._check(self.lib.mardyn_compute_forces(self.h))

    def step(self, n=1):
        self._check(self.lib.mardyn_step(self.h, int(n)))

    def get_observables(self):
        o = Observables()
        self._check(self.lib.mardyn_get_observables(self.h, C.byref(o)))
        return o.as_dict()

    def get_observable_history(self, cap=4096):
        arr = (Observables * cap)()
        n = C.c_int32()
        self._check(self.lib.mardyn_get_observable_history(self.h, cap, C.byref(n), arr))
        return [arr[k].as_dict() for k in range(n.value)]

    def get_molecules(self, out=None):
        cap = self.capacity
        res = out if out is not None else {
            "id": np.empty(cap, np.int64), "comp": np.empty(cap, np.int32),
            "r": np.empty((cap, 3)), "v": np.empty((cap, 3)), "q": np.empty((cap, 4)),
            "j": np.empty((cap, 3))}
        n = C.c_int64()
        p = {k: _out_ptr(res[k]) for k in res}
        self._check(self.lib.mardyn_get_molecules(self.h, cap, C.byref(n), p.get("id"), p.get("comp"),
                                                  p.get("r"), p.get("v"), p.get("q"), p.get("j")))
        if out is not None:
            return n.value
        return {k: x[: n.value] for k, x in res.items()}

    def get_forces(self, with_ids=False):
        cap = self.capacity
        F = np.empty((cap, 3)); tau = np.empty((cap, 3)); ids = np.empty(cap, np.int64)
        n = C.c_int64()
        self._check(self.lib.mardyn_get_forces(self.h, cap, F.ctypes.data_as(C.c_void_p),
                                               tau.ctypes.data_as(C.c_void_p), C.byref(n),
                                               ids.ctypes.data_as(C.c_void_p)))
        m = n.value
        if with_ids:
            return F[:m], tau[:m], ids[:m]
        return F[:m], tau[:m]

    def set_thermostat(self, T_target, interval=1):
        """NVT velocity rescaling every `interval` steps (reading A24); T_target = 0: NVE."""
        self._check(self.lib.mardyn_set_thermostat(self.h, float(T_target), int(interval)))

    def get_tail_corrections(self):
        """Isotropic LJ tail corrections (U_lrc, W_lrc) of the loaded system (reading A3)."""
        U, W = C.c_double(), C.c_double()
        self._check(self.lib.mardyn_get_tail_corrections(self.h, C.byref(U), C.byref(W)))
        return U.value, W.value

    # -- spatial decomposition (one context per rank; include/mardyn.h) -----
    def partition(self, r):
        """k-d partition from the global positions (mardyn_partition)."""
        ra = np.ascontiguousarray(r, dtype=np.float64)
        self._check(self.lib.mardyn_partition(self.h, len(ra), ra.ctypes.data_as(C.c_void_p)))

    def set_partition(self, boxes):
        b = np.ascontiguousarray(np.asarray(boxes, dtype=np.int32).reshape(self.nranks, 6))
        self._check(self.lib.mardyn_set_partition(self.h, b.ctypes.data_as(C.c_void_p)))

    def get_partition(self):
        """Current boxes (p, 2, 3): [lo, hi] cell ranges in (x, y, z)."""
        b = np.empty((self.nranks, 6), dtype=np.int32)
        self._check(self.lib.mardyn_get_partition(self.h, b.ctypes.data_as(C.c_void_p)))
        return b.reshape(self.nranks, 2, 3)

    def dd_counts(self, r):
        """Owned + halo molecules of every rank under the current partition."""
        ra = np.ascontiguousarray(r, dtype=np.float64)
        out = np.zeros(max(self.nranks, 1), dtype=np.int64)
        self._check(self.lib.mardyn_dd_counts(self.h, len(ra), ra.ctypes.data_as(C.c_void_p),
                                              out.ctypes.data_as(C.c_void_p)))
        return out

    def rebalance(self):
        self._check(self.lib.mardyn_rebalance(self.h))

    def set_cost_model(self, model):
        """Per-cell load of the k-d tree: 0 = Eq. 6 (default), 1 = molecule count."""
        self._check(self.lib.mardyn_set_cost_model(self.h, int(model)))

    def _n(self):
        n = C.c_int64()
        self._check(self.lib.mardyn_get_molecules(self.h, self.capacity, C.byref(n), None, None, None,
                                                  None, None, None))
        return n.value

    def get_raw(self):
        cap = self.capacity
        g = self.get_grid()
        u = np.empty((cap, 3), np.uint32)
        cell = np.empty(cap, np.int32)
        cnt = np.empty(int(np.prod(g["ncell"])), np.int32)
        self._check(self.lib.mardyn_get_raw(self.h, cap, u.ctypes.data_as(C.c_void_p),
                                            cell.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p)))
        n = self._n()
        return u[:n], cell[:n], cnt

    def last_step_timing(self):
        t = C.c_double(); f = C.c_double(); nl = C.c_int32()
        self._check(self.lib.mardyn_last_step_timing(self.h, C.byref(t), C.byref(f), C.byref(nl)))
        return {"total_ms": t.value, "force_ms": f.value, "force_launches": nl.value}

    def set_profiling(self, on):
        self._check(self.lib.mardyn_set_profiling(self.h, int(bool(on))))

    def launch_count(self):
        return int(self.lib.mardyn_launch_count(self.h))


def lj_tail(components, counts, volume, cutoff, eta=None):
    """Isotropic LJ tail corrections (U_lrc, W_lrc) for molecule counts per
    component in a volume (mardyn_lj_tail; host code, no GPU needed)."""
    lib = load_library()
    arr, keep = _components(components)
    c = np.ascontiguousarray(counts, dtype=np.int64)
    e = None if eta is None else np.ascontiguousarray(eta, dtype=np.float64)
    U, W = C.c_double(), C.c_double()
    rc = lib.mardyn_lj_tail(arr, len(components), None if e is None else e.ctypes.data_as(C.c_void_p),
                            c.ctypes.data_as(C.c_void_p), float(volume), float(cutoff), C.byref(U), C.byref(W))
    if rc:
        raise MardynError(rc, "lj_tail")
    return U.value, W.value


# host-side decomposition (no GPU needed)
def cell_cost(counts):
    """Eq. 6 per cell; counts is an (nz, ny, nx) int array (x fastest)."""
    lib = load_library()
    c = np.ascontiguousarray(counts, dtype=np.int32)
    nz, ny, nx = c.shape
    out = np.empty(c.shape, dtype=np.float64)
    rc = lib.mardyn_cell_cost(c.ctypes.data_as(C.c_void_p), nx, ny, nz, out.ctypes.data_as(C.c_void_p))
    if rc:
        raise MardynError(rc, "cell_cost")
    return out


def kd_decompose(cost, p):
    """k-d tree decomposition of an (nz, ny, nx) cost array into p boxes:
    returns (boxes (p, 2, 3) [lo, hi] in (x, y, z), loads (p,))."""
    lib = load_library()
    c = np.ascontiguousarray(cost, dtype=np.float64)
    nz, ny, nx = c.shape
    boxes = np.empty((p, 6), dtype=np.int32)
    loads = np.empty(p, dtype=np.float64)
    rc = lib.mardyn_kd_decompose(c.ctypes.data_as(C.c_void_p), nx, ny, nz, int(p),
                                 boxes.ctypes.data_as(C.c_void_p), loads.ctypes.data_as(C.c_void_p))
    if rc:
        raise MardynError(rc, "kd_decompose: 2-cell constraint cannot be met")
    return boxes.reshape(p, 2, 3), loads


def grid_counts(box, cutoff, r):
    """Molecules per cell (nz, ny, nx) of the A12 lattice (mardyn_grid_counts; host)."""
    lib = load_library()
    b = (C.c_double * 3)(*[float(x) for x in box])
    ra = np.ascontiguousarray(r, dtype=np.float64).reshape(-1, 3)
    nc = np.zeros(3, np.int32)
    rc = lib.mardyn_grid_counts(b, float(cutoff), len(ra), ra.ctypes.data_as(C.c_void_p),
                                nc.ctypes.data_as(C.c_void_p), None)
    if rc:
        raise MardynError(rc, "grid_counts")
    out = np.zeros(int(np.prod(nc)), np.int32)
    lib.mardyn_grid_counts(b, float(cutoff), len(ra), ra.ctypes.data_as(C.c_void_p), nc.ctypes.data_as(C.c_void_p),
                           out.ctypes.data_as(C.c_void_p))
    return out.reshape(nc[2], nc[1], nc[0])


def kd_partition(box, cutoff, r, p):
    """k-d partition of positions r into p boxes (mardyn_kd_partition; host):
    (boxes (p, 2, 3), loads (p,))."""
    lib = load_library()
    b = (C.c_double * 3)(*[float(x) for x in box])
    ra = np.ascontiguousarray(r, dtype=np.float64).reshape(-1, 3)
    boxes = np.empty((p, 6), np.int32)
    loads = np.empty(p)
    rc = lib.mardyn_kd_partition(b, float(cutoff), len(ra), ra.ctypes.data_as(C.c_void_p), int(p),
                                 boxes.ctypes.data_as(C.c_void_p), loads.ctypes.data_as(C.c_void_p))
    if rc:
        raise MardynError(rc, "kd_partition")
    return boxes.reshape(p, 2, 3), loads


def broadcast_unique_id(dist):
    """Rank 0's NCCL unique id (mardyn_nccl_unique_id) on every rank of the default
    torch.distributed group (the 128 bytes SURVEY §8(b) has the caller broadcast)."""
    obj = [nccl_unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def nccl_unique_id():
    """128-byte NCCL unique id (mardyn_nccl_unique_id; rank 0 calls it, the caller
    broadcasts it)."""
    lib = load_library()
    buf = C.create_string_buffer(128)
    rc = lib.mardyn_nccl_unique_id(buf)
    if rc:
        raise MardynError(rc, "nccl_unique_id: NCCL unavailable")
    return bytes(buf.raw)


class DecomposedRun:
    """p spatial subdomains (k-d tree, §4) stepping together.  All of the
    method runs in the library (include/mardyn.h): the partition, the per-step halo
    exchange and migration, the periodic rebalance and the global observables;
    this class only creates the ranks, sizes their workspaces and steps them.

    transport = "loopback": all ranks in this process on one device
    (mardyn_create_loopback; the single-GPU correctness path).
    transport = "nccl": one rank per process / GPU (mardyn_create_distributed;
    the NCCL unique id travels by torch.distributed.broadcast_object_list)."""

    def __init__(self, system, nranks, transport="loopback", rank=None, eta=None, boxes=None, stream=None,
                 rebalance_interval=0, headroom=1.5, cost_model=0):
        import torch
        self.torch = torch
        self.system, self.nranks, self.transport = system, int(nranks), transport
        args = (system["box"], system["rc"], system["components"], system["dt"])
        kw = dict(eps_rf=system.get("eps_rf", math.inf), lj_shift=system.get("lj_shift", 1), eta=eta,
                  stream=stream, rebalance_interval=rebalance_interval)
        if transport == "loopback":
            self.ctxs = Context.loopback(*args, self.nranks, **kw)
            self.rank = None
        else:
            import torch.distributed as dist
            uid = broadcast_unique_id(dist)
            self.ctxs = [Context.distributed(*args, uid, rank, self.nranks, **kw)]
            self.rank = int(rank)
        self.lead = self.ctxs[0]
        self.stream = self.lead.stream
        r = system["r"]
        self.lead.set_cost_model(cost_model)
        for c in self.ctxs:
            if boxes is None:
                c.partition(r)
            else:
                c.set_partition(np.asarray(boxes).reshape(self.nranks, 6) if np.asarray(boxes).ndim != 2
                                else boxes)
        # workspace: owned + halo of the most loaded rank (the library counts them), with
        # headroom for migration and for a rebalance that moves load between ranks
        cap = int(headroom * int(self.lead.dd_counts(r).max())) + 4096
        for c in self.ctxs:
            c.reserve(cap)
            c.set_molecules(r, system["v"], comp=system["comp"], q=system["q"], j=system["j"], id=system["id"],
                            half_step=0)

    @property
    def boxes(self):
        return self.lead.get_partition()

    def step(self, n=1):
        self.lead.step(n)

    def rebalance(self):
        self.lead.rebalance()
        return self.boxes

    def observables(self):
        return self.lead.get_observables()

    def observable_history(self, cap=4096):
        return self.lead.get_observable_history(cap)

    def compute_forces(self):
        self.lead.compute_forces()

    def owned_counts(self):
        """Owned molecules per local rank."""
        return [c._n() for c in self.ctxs]

    def molecules(self):
        """Owned molecules of the local ranks, merged and ordered by id."""
        parts = [c.get_molecules() for c in self.ctxs]
        ids = np.concatenate([p["id"] for p in parts])
        order = np.argsort(ids)
        return {k: np.concatenate([p[k] for p in parts])[order] for k in parts[0]}

    def forces(self):
        parts = [c.get_forces(with_ids=True) for c in self.ctxs]
        ids = np.concatenate([p[2] for p in parts])
        order = np.argsort(ids)
        return (np.concatenate([p[0] for p in parts])[order], np.concatenate([p[1] for p in parts])[order],
                ids[order])


# module-level aliases with the C names
def mardyn_create(box, cutoff, components, dt, **kw):
    return Context(box, cutoff, components, dt, **kw)


def from_system(system, stream=None, capacity=None, eta=None):
    """Context + molecules of a scenarios system dict (on-step v, j: A8)."""
    ctx = Context(system["box"], system["rc"], system["components"], system["dt"],
                  eps_rf=system.get("eps_rf", math.inf), lj_shift=system.get("lj_shift", 1),
                  eta=eta, capacity=capacity or len(system["r"]), stream=stream)
    ctx.set_molecules(system["r"], system["v"], comp=system["comp"], q=system["q"], j=system["j"],
                      id=system["id"], half_step=0)
    return ctx
