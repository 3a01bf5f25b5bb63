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
           "mardyn_set_decomposition", "mardyn_dd_begin_step", "mardyn_dd_buffers", "mardyn_dd_end_step",
           "mardyn_dd_set_segment", "mardyn_dd_set_peer_segments", "mardyn_dd_device_counts",
           "mardyn_dd_set_peer_targets",
           "mardyn_dd_begin_step_async",
           "mardyn_dd_end_step_async",
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
                ("eta", C.POINTER(C.c_double)), ("cuda_stream", C.c_void_p)]


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
    lib.mardyn_set_decomposition.argtypes = [vp, C.c_int32, C.c_int32, vp, C.c_double]
    lib.mardyn_set_thermostat.argtypes = [vp, C.c_double, C.c_int32]
    lib.mardyn_lj_tail.argtypes = [P(Component), C.c_int32, vp, vp, C.c_double, C.c_double, P(C.c_double),
                                   P(C.c_double)]
    lib.mardyn_get_tail_corrections.argtypes = [vp, P(C.c_double), P(C.c_double)]
    lib.mardyn_dd_begin_step.argtypes = [vp, vp]
    lib.mardyn_dd_buffers.argtypes = [vp, P(vp), P(C.c_int64), P(vp), P(C.c_int64), P(C.c_int32)]
    lib.mardyn_dd_end_step.argtypes = [vp, C.c_int64]
    lib.mardyn_dd_set_segment.argtypes = [vp, C.c_int64]
    lib.mardyn_dd_set_peer_segments.argtypes = [vp, vp, vp]
    lib.mardyn_dd_device_counts.argtypes = [vp, P(vp), P(vp)]
    lib.mardyn_dd_set_peer_targets.argtypes = [vp, vp, vp]
    lib.mardyn_dd_begin_step_async.argtypes = [vp]
    lib.mardyn_dd_end_step_async.argtypes = [vp]
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
                 capacity=None, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("mardyn needs a CUDA device (there is no CPU fallback)")
        self.lib = load_library()
        self.torch = torch
        self.stream = stream if stream is not None else torch.cuda.Stream()
        comps, self._keep = _components(components)
        self._eta = None if eta is None else np.ascontiguousarray(eta, dtype=np.float64)
        opt = Options()
        opt.dt = float(dt)
        opt.eps_rf = float(eps_rf)
        opt.lj_shift = int(lj_shift)
        opt.eta = None if self._eta is None else self._eta.ctypes.data_as(C.POINTER(C.c_double))
        opt.cuda_stream = C.c_void_p(self.stream.cuda_stream)
        box_a = (C.c_double * 3)(*[float(x) for x in box])
        h = C.c_void_p()
        rc = self.lib.mardyn_create(box_a, float(cutoff), comps, len(components), C.byref(opt), C.byref(h))
        self.h = h
        self.ws = None
        self.capacity = 0
        self._check(rc)
        if capacity is not None:
            self.reserve(capacity)

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

    # -- spatial decomposition (one context per rank) ----------------------
    def set_thermostat(self, T_target, interval=1):
        """NVT velocity rescaling every `interval` steps (reading A24); T_target = 0: NVE."""
        self._check(self.lib.mardyn_set_thermostat(self.h, float(T_target), int(interval)))

    def get_tail_corrections(self):
        """Isotropic LJ tail corrections (U_lrc, W_lrc) of the loaded system (reading A3)."""
        U, W = C.c_double(), C.c_double()
        self._check(self.lib.mardyn_get_tail_corrections(self.h, C.byref(U), C.byref(W)))
        return U.value, W.value

    def set_decomposition(self, rank, nranks, boxes, ndof_global):
        b = np.ascontiguousarray(np.asarray(boxes, dtype=np.int32).reshape(nranks, 6))
        self._dd_boxes = b
        self._check(self.lib.mardyn_set_decomposition(self.h, int(rank), int(nranks),
                                                      b.ctypes.data_as(C.c_void_p), float(ndof_global)))
        self.rank, self.nranks = int(rank), int(nranks)

    def dd_begin_step(self):
        cnt = np.zeros(self.nranks, np.int64)
        self._check(self.lib.mardyn_dd_begin_step(self.h, cnt.ctypes.data_as(C.c_void_p)))
        return cnt

    def dd_buffers(self):
        """(send tensor view [nranks, seg_cap, rec], recv tensor view [recv_cap, rec])
        as uint8 slices of the workspace tensor (zero copy)."""
        send = C.c_void_p(); seg = C.c_int64(); recv = C.c_void_p(); rcap = C.c_int64(); rb = C.c_int32()
        self._check(self.lib.mardyn_dd_buffers(self.h, C.byref(send), C.byref(seg), C.byref(recv),
                                               C.byref(rcap), C.byref(rb)))
        base = self.ws.data_ptr()
        so, ro = send.value - base, recv.value - base
        sb = self.ws[so: so + self.nranks * seg.value * rb.value].view(self.nranks, seg.value, rb.value)
        rv = self.ws[ro: ro + rcap.value * rb.value].view(rcap.value, rb.value)
        return sb, rv

    def dd_end_step(self, n_recv):
        self._check(self.lib.mardyn_dd_end_step(self.h, int(n_recv)))

    # asynchronous decomposed step (include/mardyn.h): counts stay in device memory
    def dd_set_segment(self, seg_cap):
        self._check(self.lib.mardyn_dd_set_segment(self.h, int(seg_cap)))

    def dd_set_peer_segments(self, send_caps, recv_caps):
        sc = np.ascontiguousarray(np.asarray(send_caps, dtype=np.int64))
        rc = np.ascontiguousarray(np.asarray(recv_caps, dtype=np.int64))
        self._check(self.lib.mardyn_dd_set_peer_segments(self.h, sc.ctypes.data_as(C.c_void_p),
                                                         rc.ctypes.data_as(C.c_void_p)))

    def dd_set_peer_targets(self, rec_addrs, cnt_addrs):
        """Direct puts (include/mardyn.h): device addresses, per destination rank, of this
        rank's receive segment and count entry in that rank's buffers; None: transport."""
        if rec_addrs is None:
            self._check(self.lib.mardyn_dd_set_peer_targets(self.h, None, None))
            return
        ra = np.ascontiguousarray(np.asarray(rec_addrs, dtype=np.uint64))
        ca = np.ascontiguousarray(np.asarray(cnt_addrs, dtype=np.uint64))
        self._check(self.lib.mardyn_dd_set_peer_targets(self.h, ra.ctypes.data_as(C.c_void_p),
                                                        ca.ctypes.data_as(C.c_void_p)))

    def dd_device_counts(self):
        """(send_cnt, recv_cnt): int32 [nranks] tensor views of the workspace (zero copy)."""
        sc = C.c_void_p(); rc = C.c_void_p()
        self._check(self.lib.mardyn_dd_device_counts(self.h, C.byref(sc), C.byref(rc)))
        base = self.ws.data_ptr()
        view = lambda ptr: self.ws[ptr - base: ptr - base + 4 * self.nranks].view(self.torch.int32)
        return view(sc.value), view(rc.value)

    def dd_begin_step_async(self):
        self._check(self.lib.mardyn_dd_begin_step_async(self.h))

    def dd_end_step_async(self):
        self._check(self.lib.mardyn_dd_end_step_async(self.h))

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


def system_ndof(system):
    """3 N + rotational degrees of freedom (nonzero principal moments), A9."""
    rot = np.array([sum(1 for x in c["inertia"] if x > 0) for c in system["components"]])
    return float(3 * len(system["r"]) + rot[np.asarray(system["comp"])].sum())


def global_costs(system):
    """Eq. 6 per cell of the global grid (x fastest) for the k-d tree, from
    the molecule counts per cell of edge >= rc (every rank computes the same)."""
    box = np.asarray(system["box"], float)
    n = np.floor(box / system["rc"]).astype(int)
    c = np.minimum((np.asarray(system["r"]) % box / box * n).astype(int), n - 1)
    counts = np.zeros((n[2], n[1], n[0]), np.int32)
    np.add.at(counts, (c[:, 2], c[:, 1], c[:, 0]), 1)
    return cell_cost(counts)


def peer_target_addrs(me, bases, rows, record_bytes):
    """Direct puts (include/mardyn.h mardyn_dd_set_peer_targets): device addresses, per
    destination rank d, of rank me's receive segment and count entry in d's buffers.
    bases[d]: base address of d's (symmetric) allocation; rows[d] = [receive buffer offset,
    count array offset (bytes, from bases[d]), then d's receive segment offsets (records)
    per source rank].  Loopback: bases = 0 and absolute addresses."""
    p = len(bases)
    rec = [int(bases[d]) + int(rows[d][0]) + record_bytes * int(rows[d][2 + me]) for d in range(p)]
    cnt = [int(bases[d]) + int(rows[d][1]) + 4 * me for d in range(p)]
    return rec, cnt


def exchange_records(send, cnt, recv, nranks, dist):
    """Halo/migration transport between ranks:
    send[d, :cnt[d]] goes to rank d; records from all ranks land contiguously
    in recv in source-rank order.  Counts travel first (all_to_all_single),
    then the records as grouped point-to-point send/recv (NCCL over NVLink on
    GPUs, gloo on CPU).  Returns the number of records received."""
    import torch
    dev = recv.device
    sc = torch.tensor([int(x) for x in cnt], dtype=torch.int64, device=dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc)
    rcounts = rc.cpu().tolist()
    outs, off = [], 0
    for k in rcounts:
        outs.append(recv[off: off + k])
        off += k
    me = dist.get_rank()
    # gloo moves device tensors in its collectives but not point to point: stage through host
    host = dev.type == "cuda" and dist.get_backend() != "nccl"
    ops, land = [], []
    for d in range(nranks):
        if d == me:
            if int(cnt[d]):
                outs[d].copy_(send[d][: int(cnt[d])])
            continue
        if int(cnt[d]):
            t = send[d][: int(cnt[d])].contiguous()
            ops.append(dist.P2POp(dist.isend, t.cpu() if host else t, d))
        if rcounts[d]:
            t = torch.empty(outs[d].shape, dtype=outs[d].dtype) if host else outs[d]
            land.append((outs[d], t))
            ops.append(dist.P2POp(dist.irecv, t, d))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    if host:
        for o, t in land:
            o.copy_(t)
    return off


def exchange_segments(send, send_cnt, recv, recv_cnt, nranks, dist, send_caps=None, recv_caps=None):
    """Transport of the asynchronous decomposed step (include/mardyn.h): rank r's
    send segment d lands in segment r of rank d's receive buffer, and its record
    count send_cnt[d] in recv_cnt[r] of rank d.  send / recv: [records, bytes]
    views of the exchange buffers with the segments back to back -- all of size
    seg = len(send) / nranks (uniform), or send_caps[d] / recv_caps[r] records
    (per-peer, static split sizes).  Two all-to-alls; nothing is read on the host
    (NCCL over NVLink on GPUs, gloo on CPU)."""
    dist.all_to_all_single(recv_cnt, send_cnt)
    rb = send.shape[-1]
    if send_caps is None:
        n = send.shape[0]
        dist.all_to_all_single(recv[:n].reshape(-1), send.reshape(-1))
    else:
        ns, nr = int(sum(send_caps)), int(sum(recv_caps))
        dist.all_to_all_single(recv[:nr].reshape(-1), send[:ns].reshape(-1),
                               output_split_sizes=[int(c) * rb for c in recv_caps],
                               input_split_sizes=[int(c) * rb for c in send_caps])


class DecomposedRun:
    """p spatial subdomains (k-d tree, §4) stepping together.

    transport = "loopback": all ranks' contexts live in this process on one
    device and records move by device copies (correctness path, 1 GPU).
    transport = "nccl": one rank per process/GPU, records move with
    torch.distributed all_to_all over NCCL (NVLink)."""

    def __init__(self, system, nranks, transport="loopback", rank=None, eta=None, boxes=None, stream=None,
                 rebalance_interval=0, async_exchange=True, direct=False):
        import torch
        self.torch = torch
        # one stream for every local context and the transport: the asynchronous step
        # orders the exchange after the packing and before the import by the stream alone
        self.stream = stream if stream is not None else torch.cuda.Stream()
        stream = self.stream
        self.async_exchange = bool(async_exchange)
        # device-initiated exchange: the packing kernels store the records straight into the
        # receiving contexts' buffers -- loopback: same device, ordered by the stream; NCCL
        # ranks: workspaces in symmetric memory (peer pointers over NVLink) and a device
        # barrier before the puts and before the import of every step
        self.direct = bool(direct) and self.async_exchange
        self.symm = None
        alloc = None
        if self.direct and transport != "loopback":
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm
            try:
                symm.enable_symm_mem_for_group(dist.group.WORLD.group_name)
            except Exception:
                pass
            dev = torch.device("cuda", torch.cuda.current_device())
            alloc = lambda nb: symm.empty(nb, dtype=torch.uint8, device=dev)
        self.seg_ready = False
        self.system = system
        self.nranks = nranks
        self.transport = transport
        self.rank = rank
        self.rebalance_interval = int(rebalance_interval)   # steps between re-partitions (0: static)
        self.nsteps = 0
        cost = global_costs(system)
        if boxes is None:
            boxes, loads = kd_decompose(cost, nranks)
        self.boxes = np.asarray(boxes).reshape(nranks, 2, 3)
        flat = np.concatenate([self.boxes[:, 0, :], self.boxes[:, 1, :]], axis=1)
        ndof = system_ndof(system)
        self.ndof = ndof
        ranks = range(nranks) if transport == "loopback" else [rank]
        self.ctxs = []
        for r in ranks:
            ctx = Context(system["box"], system["rc"], system["components"], system["dt"],
                          eps_rf=system.get("eps_rf", math.inf), lj_shift=system.get("lj_shift", 1), eta=eta,
                          stream=stream)
            ctx.set_decomposition(r, nranks, flat, ndof)
            # every rank takes the GLOBAL arrays in set_molecules (the library keeps the owned
            # and halo molecules), so the capacity -- which also sizes the input staging -- is
            # at least the global count; twice that holds owned + halo + received records of
            # small boxes whose halo is as large as the box; the asynchronous step's
            # capacity-wide grids exit early past the rank's molecules
            ctx.reserve(2 * len(system["r"]), alloc=alloc)
            if alloc is not None:
                import torch.distributed as dist
                import torch.distributed._symmetric_memory as symm
                self.symm = symm.rendezvous(ctx.ws, dist.group.WORLD)
            ctx.set_molecules(system["r"], system["v"], comp=system["comp"], q=system["q"], j=system["j"],
                              id=system["id"], half_step=0)
            self.ctxs.append(ctx)
        self.bufs = [c.dd_buffers() for c in self.ctxs]
        self.seg_max = int(self.bufs[0][0].shape[1])

    def gather_molecules(self):
        """All owned molecules of all ranks (v, j at t - dt/2), ordered by id."""
        if self.transport == "loopback":
            return self.molecules()
        import torch.distributed as dist
        parts = [None] * self.nranks
        dist.all_gather_object(parts, self.ctxs[0].get_molecules())
        ids = np.concatenate([p["id"] for p in parts])
        order = np.argsort(ids)
        return {k: np.concatenate([p[k] for p in parts])[order] for k in parts[0]}

    def rebalance(self, boxes=None):
        """Re-partition from the current cell counts (Eq. 6 cost of reading A19,
        k-d tree with alternating axes and minimum-imbalance planes)
        and reload every rank's owned + halo molecules (exact resume).  Returns
        the new boxes."""
        m = self.gather_molecules()
        now = dict(self.system)
        now["r"], now["comp"] = m["r"], m["comp"]
        if boxes is None:
            boxes, _ = kd_decompose(global_costs(now), self.nranks)
        self.boxes = np.asarray(boxes).reshape(self.nranks, 2, 3)
        flat = np.concatenate([self.boxes[:, 0, :], self.boxes[:, 1, :]], axis=1)
        ranks = range(self.nranks) if self.transport == "loopback" else [self.rank]
        for r, ctx in zip(ranks, self.ctxs):
            ctx.set_decomposition(r, self.nranks, flat, self.ndof)
            ctx.set_molecules(m["r"], m["v"], comp=m["comp"], q=m["q"], j=m["j"], id=m["id"], half_step=1)
            ctx.dd_set_segment(int(ctx.dd_buffers()[0].shape[1]))
        self.bufs = [c.dd_buffers() for c in self.ctxs]
        self.seg_max = min(int(b[0].shape[1]) for b in self.bufs)
        self.seg_ready = False                       # re-size the exchange segments for the new boxes
        return self.boxes

    def owned_counts(self):
        """Owned molecules per rank (load balance check)."""
        if self.transport == "loopback":
            return [len(c.get_molecules()["id"]) for c in self.ctxs]
        import torch.distributed as dist
        parts = [None] * self.nranks
        dist.all_gather_object(parts, len(self.ctxs[0].get_molecules()["id"]))
        return parts

    def step(self, n=1):
        """n time steps of all local ranks.  The first step after construction or a
        rebalance runs with host-side record counts and sizes the exchange segments
        (twice the largest count + 1024 records); the following steps run
        asynchronously (no host synchronisation: counts and records move between
        ranks as two all-to-alls with equal splits, see include/mardyn.h)."""
        with self.torch.cuda.stream(self.stream):
            for _ in range(n):
                if self.rebalance_interval and self.nsteps and self.nsteps % self.rebalance_interval == 0:
                    self.rebalance()
                self.nsteps += 1
                if self.async_exchange and self.seg_ready:
                    self._step_async()
                    continue
                counts = [c.dd_begin_step() for c in self.ctxs]
                if self.transport == "loopback":
                    for dst, cd in enumerate(self.ctxs):
                        recv = self.bufs[dst][1]
                        off = 0
                        for src in range(self.nranks):
                            k = int(counts[src][dst])
                            if k:
                                recv[off: off + k].copy_(self.bufs[src][0][dst, :k])
                                off += k
                        cd.dd_end_step(off)
                else:
                    self._nccl_exchange(counts[0])
                if self.async_exchange:
                    self._size_segments(counts)

    def _size_segments(self, counts):
        """Per-peer exchange segments from the first step's record counts: twice the
        count + 1024 records (face neighbours send far more than edge or corner ones);
        uniform segments if the per-peer ones do not fit the buffers."""
        torch, p = self.torch, self.nranks
        cap = lambda c: ((2 * int(c) + 1024 + 255) // 256) * 256
        send_caps = [[cap(c) for c in cnt] for cnt in counts]          # per local rank, per destination
        if self.transport == "loopback":
            ranks = list(range(p))
            recv_caps = [[send_caps[src][dst] for src in range(p)] for dst in range(p)]
        else:
            import torch.distributed as dist
            ranks = [self.rank]
            t = torch.tensor(send_caps[0], dtype=torch.int64, device="cuda")
            r = torch.empty_like(t)
            dist.all_to_all_single(r, t)
            recv_caps = [r.tolist()]
        recv_cap = int(self.bufs[0][1].shape[0])
        fits = all(sum(sc) <= self.seg_max * p and sum(rc) <= recv_cap for sc, rc in zip(send_caps, recv_caps))
        if self.transport != "loopback":
            import torch.distributed as dist
            t = torch.tensor([0 if fits else 1], dtype=torch.int32, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            fits = int(t.item()) == 0
        if fits:
            for c, sc, rc in zip(self.ctxs, send_caps, recv_caps):
                c.dd_set_peer_segments(sc, rc)
            self.send_caps, self.recv_caps = send_caps, recv_caps
        else:
            big = max(max(sc) for sc in send_caps)
            if self.transport != "loopback":
                t = torch.tensor([big], dtype=torch.int64, device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                big = int(t.item())
            seg = min(self.seg_max, recv_cap // p, big)
            for c in self.ctxs:
                c.dd_set_segment(seg)
            self.send_caps = [[seg] * p for _ in self.ctxs]
            self.recv_caps = [[seg] * p for _ in self.ctxs]
        self.bufs = [c.dd_buffers() for c in self.ctxs]
        self.flat = [(sb.reshape(-1, sb.shape[-1]), rv) for sb, rv in self.bufs]   # [records, bytes] views
        self.cnts = [c.dd_device_counts() for c in self.ctxs]
        self.puts = False
        if self.direct:
            rb = int(self.flat[0][1].shape[-1])
            offs = lambda caps: [int(sum(caps[:r])) for r in range(p)]
            if self.transport == "loopback":
                rows = [[self.flat[d][1].data_ptr(), self.cnts[d][1].data_ptr()] + offs(self.recv_caps[d])
                        for d in range(p)]
                for src, c in enumerate(self.ctxs):
                    c.dd_set_peer_targets(*peer_target_addrs(src, [0] * p, rows, rb))
            else:
                import torch.distributed as dist
                bases = list(self.symm.buffer_ptrs)
                mine = [self.flat[0][1].data_ptr() - bases[self.rank],
                        self.cnts[0][1].data_ptr() - bases[self.rank]] + offs(self.recv_caps[0])
                t = torch.tensor(mine, dtype=torch.int64, device="cuda")
                allt = [torch.empty_like(t) for _ in range(p)]
                dist.all_gather(allt, t)
                rows = [x.tolist() for x in allt]
                self.ctxs[0].dd_set_peer_targets(*peer_target_addrs(self.rank, bases, rows, rb))
            self.puts = True
        self.seg_ready = True

    def _step_async(self):
        p = self.nranks
        if self.puts and self.symm is not None:
            self.symm.barrier(channel=0)       # every rank's last import done: its buffers are free
        for c in self.ctxs:
            c.dd_begin_step_async()
        if self.puts:
            # records and counts already stored by the packing kernels (peers: after the barrier)
            if self.symm is not None:
                self.symm.barrier(channel=0)
        elif self.transport == "loopback":
            soff = [np.concatenate([[0], np.cumsum(sc)[:-1]]) for sc in self.send_caps]
            roff = [np.concatenate([[0], np.cumsum(rc)[:-1]]) for rc in self.recv_caps]
            for dst in range(p):
                rcnt = self.cnts[dst][1]
                for src in range(p):
                    c = int(self.send_caps[src][dst])
                    a, b = int(roff[dst][src]), int(soff[src][dst])
                    self.flat[dst][1][a: a + c].copy_(self.flat[src][0][b: b + c])
                    rcnt[src: src + 1].copy_(self.cnts[src][0][dst: dst + 1])
        else:
            import torch.distributed as dist
            send, recv = self.flat[0]
            scnt, rcnt = self.cnts[0]
            try:
                exchange_segments(send, scnt, recv, rcnt, p, dist, self.send_caps[0], self.recv_caps[0])
            except RuntimeError:
                # a backend without these all-to-alls: finish this step with host-side
                # counts and point-to-point records, and stay on that path
                self.async_exchange = False
                sc = self.send_caps[0]
                off = np.concatenate([[0], np.cumsum(sc)[:-1]])
                segs = [send[int(off[d]): int(off[d]) + int(sc[d])] for d in range(p)]
                cnt = [min(int(x), int(sc[d])) for d, x in enumerate(scnt.cpu().tolist())]   # overflow: flagged
                n = exchange_records(segs, cnt, recv, p, dist)
                self.ctxs[0].dd_end_step(n)
                return
        for c in self.ctxs:
            c.dd_end_step_async()

    def _nccl_exchange(self, cnt):
        import torch.distributed as dist
        ctx = self.ctxs[0]
        send, recv = self.bufs[0]
        n = exchange_records(send, cnt, recv, self.nranks, dist)
        ctx.dd_end_step(n)

    def observables(self):
        keys = ("U_pot", "virial", "T", "E_kin_trans", "E_kin_rot", "n_pairs", "n_candidates")
        if self.transport == "loopback":
            parts = [c.get_observables() for c in self.ctxs]
        else:
            import torch.distributed as dist
            parts = [None] * self.nranks
            dist.all_gather_object(parts, self.ctxs[0].get_observables())
        out = dict(parts[0])
        for k in keys:
            out[k] = sum(p[k] for p in parts)        # rank order: deterministic
        out["n_pairs"] //= 2                         # ranks report ordered pairs of owned molecules
        return out

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
