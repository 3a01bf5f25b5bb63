"""The NCCL-API stand-in of the one-GPU multi-process tests (tests/nccl_shim.c), checked on
the host (MDSHIM_HOST=1: buffers are host memory, no CUDA) with three processes before it
is trusted to carry the library's exchange in tests/test_gpu_nccl_shim.py: grouped
send / recv matched in issue order per pair, sends and receives of one group in any order
without deadlock, all-reduce (sum, max) and all-gather in rank order, many rounds (the
sequence numbers and the file clean-up)."""
import ctypes as C
import multiprocessing as mp
import os

import numpy as np
import pytest

from nccl_shim_util import build_shim

NCCL_CHAR, NCCL_INT32, NCCL_INT64, NCCL_DOUBLE = 0, 2, 4, 8
NCCL_SUM, NCCL_MAX = 0, 2


def _worker(rank, world, shim, uid_path, q):
    try:
        os.environ["MDSHIM_HOST"] = "1"
        os.environ["MDSHIM_TIMEOUT_S"] = "60"
        L = C.CDLL(shim)
        if rank == 0:
            uid = C.create_string_buffer(128)
            assert L.ncclGetUniqueId(uid) == 0
            with open(uid_path + ".tmp", "wb") as f:
                f.write(uid.raw)
            os.rename(uid_path + ".tmp", uid_path)
        while not os.path.exists(uid_path):
            pass
        uid = C.create_string_buffer(open(uid_path, "rb").read(), 128)

        class Uid(C.Structure):
            _fields_ = [("internal", C.c_char * 128)]
        u = Uid()
        C.memmove(C.byref(u), uid, 128)
        comm = C.c_void_p()
        assert L.ncclCommInitRank(C.byref(comm), world, u, rank) == 0
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)
        for it in range(6):
            # every rank sends (rank + 1 + it + 3 d) int64 values to each peer d, receives
            # posted before sends for odd ranks (order inside a group must not matter)
            sends, recvs = {}, {}
            for d in range(world):
                if d == rank:
                    continue
                sends[d] = np.arange(rank + 1 + it + 3 * d, dtype=np.int64) + 1000 * rank + 100 * it
                recvs[d] = np.full(d + 1 + it + 3 * rank, -1, np.int64)
            assert L.ncclGroupStart() == 0
            peers = [d for d in range(world) if d != rank]
            for d in (reversed(peers) if rank % 2 else peers):
                if rank % 2:
                    assert L.ncclRecv(ptr(recvs[d]), C.c_size_t(recvs[d].size), NCCL_INT64, d, comm, None) == 0
                    assert L.ncclSend(ptr(sends[d]), C.c_size_t(sends[d].size), NCCL_INT64, d, comm, None) == 0
                else:
                    assert L.ncclSend(ptr(sends[d]), C.c_size_t(sends[d].size), NCCL_INT64, d, comm, None) == 0
                    assert L.ncclRecv(ptr(recvs[d]), C.c_size_t(recvs[d].size), NCCL_INT64, d, comm, None) == 0
            assert L.ncclGroupEnd() == 0
            for d, r in recvs.items():
                assert np.array_equal(r, np.arange(d + 1 + it + 3 * rank, dtype=np.int64) + 1000 * d + 100 * it)
            # two messages to one peer in a row, outside a group: matched in issue order
            nxt, prv = (rank + 1) % world, (rank - 1) % world
            a1 = np.array([rank, it, 1], np.int32)
            a2 = np.array([rank, it, 2, 7], np.int32)
            b1, b2 = np.zeros(3, np.int32), np.zeros(4, np.int32)
            assert L.ncclGroupStart() == 0
            L.ncclSend(ptr(a1), C.c_size_t(3), NCCL_INT32, nxt, comm, None)
            L.ncclSend(ptr(a2), C.c_size_t(4), NCCL_INT32, nxt, comm, None)
            L.ncclRecv(ptr(b1), C.c_size_t(3), NCCL_INT32, prv, comm, None)
            L.ncclRecv(ptr(b2), C.c_size_t(4), NCCL_INT32, prv, comm, None)
            assert L.ncclGroupEnd() == 0
            assert list(b1) == [prv, it, 1] and list(b2) == [prv, it, 2, 7]
            # all-reduce: in place, int32 max and double sum; all-gather of int64 rows
            f = np.array([rank == it % world], np.int32)
            assert L.ncclAllReduce(ptr(f), ptr(f), C.c_size_t(1), NCCL_INT32, NCCL_MAX, comm, None) == 0
            assert f[0] == 1
            x = np.array([0.1 * (rank + 1), rank + it], np.float64)
            assert L.ncclAllReduce(ptr(x), ptr(x), C.c_size_t(2), NCCL_DOUBLE, NCCL_SUM, comm, None) == 0
            assert x[0] == ((0.1 * 1 + 0.1 * 2) + 0.1 * 3)          # rank order
            assert x[1] == sum(r + it for r in range(world))
            row = np.array([rank, it, rank * it], np.int64)
            allr = np.zeros(3 * world, np.int64)
            assert L.ncclAllGather(ptr(row), ptr(allr), C.c_size_t(3), NCCL_INT64, comm, None) == 0
            assert allr.reshape(world, 3).tolist() == [[r, it, r * it] for r in range(world)]
        assert L.ncclCommDestroy(comm) == 0
        q.put((rank, "ok"))
    except BaseException as e:          # reported to the parent
        q.put((rank, repr(e)))


def test_shim_semantics_three_processes(tmp_path, monkeypatch):
    shim = build_shim(tmp_path)
    monkeypatch.setenv("MDSHIM_DIR", str(tmp_path))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 3
    ps = [ctx.Process(target=_worker, args=(r, world, shim, str(tmp_path / "uid"), q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res
    d = [x for x in os.listdir(tmp_path) if x.startswith("mdshim_")][0]
    left = os.listdir(tmp_path / d)
    assert not any(x.startswith("p") for x in left), left       # every message consumed once
