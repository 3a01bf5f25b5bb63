"""Host-side load model (Eq. 6) and k-d tree decomposition
(>= 2 cells per subvolume P:213) of the C ABI, without a GPU;
plus a world_size-2 gloo run in which each rank bins its own molecules and
an all-reduce of the per-cell counts gives every rank the same tree."""
import os

import numpy as np
import pytest

import scenarios as S
from paper_1408_4599_b200 import mardyn as M


def brute_cost(counts):
    nz, ny, nx = counts.shape
    out = np.zeros(counts.shape)
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                s = 0
                for dz in (-1, 0, 1):
                    for dy in (-1, 0, 1):
                        for dx in (-1, 0, 1):
                            if dx or dy or dz:
                                s += counts[(z + dz) % nz, (y + dy) % ny, (x + dx) % nx]
                Ni = counts[z, y, x]
                out[z, y, x] = 0.5 * Ni * (Ni + s)
    return out


def test_eq6_examples():
    """SPEC S:377-379 examples of Eq. 6 and a brute-force evaluation."""
    c = np.zeros((3, 3, 3), np.int32)
    c[1, 1, 1] = 3
    c[0, 0, 0] = 7                      # the only populated neighbour
    cost = M.cell_cost(c)
    assert cost[1, 1, 1] == pytest.approx(1.5 * (3 + 7))
    c2 = np.zeros((4, 4, 4), np.int32)
    c2[2, 2, 2] = 2
    assert M.cell_cost(c2)[2, 2, 2] == pytest.approx(2.0)
    assert M.cell_cost(c2)[0, 0, 0] == 0.0
    rng = np.random.default_rng(0)
    c3 = rng.integers(0, 20, size=(4, 5, 6)).astype(np.int32)
    assert np.allclose(M.cell_cost(c3), brute_cost(c3))


def profile_cost(profile, axis_len=(4, 4)):
    """A cost field along x with the given 1-D profile (constant in y, z)."""
    p = np.asarray(profile, float)
    return np.broadcast_to(p[None, None, :] / (axis_len[0] * axis_len[1]),
                           (axis_len[1], axis_len[0], len(p))).copy()


@pytest.mark.parametrize("profile,cut", [([4, 4, 4, 4], 2), ([10, 1, 1, 1, 1, 1, 1, 2], 2),
                                         ([1, 1, 1, 1, 1, 1], 3)])
def test_best_split_examples(profile, cut):
    """minimum-imbalance plane with >= 2 cells per side."""
    boxes, loads = M.kd_decompose(profile_cost(profile), 2)
    assert boxes[0, 1, 0] == cut and boxes[1, 0, 0] == cut


def partition_ok(boxes, shape):
    nz, ny, nx = shape
    owner = -np.ones(shape, int)
    for r, (lo, hi) in enumerate(boxes):
        assert np.all(hi - lo >= 2)
        sub = owner[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        assert np.all(sub == -1)
        sub[...] = r
    return np.all(owner >= 0)


def test_uniform_octants_and_trivial():
    boxes, loads = M.kd_decompose(np.ones((8, 8, 8)), 8)
    assert all(np.all(hi - lo == 4) for lo, hi in boxes)
    assert np.allclose(loads, 64)
    boxes, loads = M.kd_decompose(np.ones((5, 6, 7)), 1)
    assert boxes[0].tolist() == [[0, 0, 0], [7, 6, 5]]


def test_minimum_imbalance_is_optimal():
    """Exhaustive check of the first cut on random profiles."""
    rng = np.random.default_rng(1)
    for _ in range(20):
        n = int(rng.integers(4, 20))
        prof = rng.uniform(0, 10, size=n)
        boxes, _ = M.kd_decompose(profile_cost(prof), 2)
        k = boxes[0, 1, 0]
        imb = lambda kk: abs(prof[:kk].sum() - prof[kk:].sum())
        assert imb(k) <= min(imb(kk) for kk in range(2, n - 1)) + 1e-9


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8])
def test_partition_invariants(p):
    rng = np.random.default_rng(p)
    cost = rng.uniform(0, 1, size=(10, 11, 12))
    boxes, loads = M.kd_decompose(cost, p)
    assert partition_ok(boxes, cost.shape)
    assert loads.sum() == pytest.approx(cost.sum())


def test_overdecomposition_rejected():
    with pytest.raises(M.MardynError):
        M.kd_decompose(np.ones((3, 3, 3)), 2)


def test_slab_and_droplet_balance():
    """Heterogeneous systems: the k-d tree balances a dense block
    better than equal volumes."""
    c = np.ones((16, 16, 16))
    c[2:6, 3:7, 9:13] = 400.0           # off-centre droplet
    boxes, loads = M.kd_decompose(c, 4)
    kd = loads.max() / loads.mean()
    eq = max(c[:, :, :8].reshape(16, 16, 8)[:8].sum(), c[:8, :, 8:].sum(), c[8:, :, :8].sum(),
             c[8:, :, 8:].sum()) / (c.sum() / 4)
    assert kd < eq
    # config-4-like slab in z: the tree does not cut it into unequal z-slabs
    s = np.ones((30, 10, 10)) * 0.01
    s[10:20] = 1.0
    boxes, loads = M.kd_decompose(s, 8)
    assert loads.max() / loads.mean() < 1.1


def _rank_main(rank, world, port, result):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    s = S.config("c4s")
    # each rank owns half of the molecules and bins them (cells of edge >= rc)
    n = np.floor(s["box"] / s["rc"]).astype(int)
    mine = np.arange(len(s["r"]))[rank::world]
    c = np.minimum((s["r"][mine] / s["box"] * n).astype(int), n - 1)
    counts = np.zeros((n[2], n[1], n[0]), np.int64)
    np.add.at(counts, (c[:, 2], c[:, 1], c[:, 0]), 1)
    t = torch.from_numpy(counts)
    dist.all_reduce(t)                                # per-cell counts of all ranks
    cost = M.cell_cost(t.numpy().astype(np.int32))
    boxes, loads = M.kd_decompose(cost, 4)
    gathered = [None] * world
    dist.all_gather_object(gathered, boxes.tolist())
    result[rank] = (gathered, int(t.sum()), float(loads.max() / loads.mean()))
    dist.destroy_process_group()


def test_gloo_two_ranks_agree():
    import torch.multiprocessing as mp
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_rank_main, args=(2, port, result), nprocs=2, join=True)
    g0, n0, imb0 = result[0]
    g1, n1, imb1 = result[1]
    assert g0[0] == g0[1] == g1[0] == g1[1]          # every rank builds the same tree
    assert n0 == n1 == len(S.config("c4s")["r"])
    assert imb0 == imb1 and imb0 < 1.2


def _xchg_main(rank, world, port, result):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rec = 64
    seg = 8
    send = torch.zeros((world, seg, rec), dtype=torch.uint8)
    cnt = [(rank + d) % 3 + 1 for d in range(world)]          # records for rank d
    for d in range(world):
        for k in range(cnt[d]):
            send[d, k, 0] = rank
            send[d, k, 1] = d
            send[d, k, 2] = k
    recv = torch.zeros((world * seg, rec), dtype=torch.uint8)
    n = M.exchange_records(send, cnt, recv, world, dist)
    result[rank] = (n, recv[:n, :3].tolist())
    dist.destroy_process_group()


def test_gloo_exchange_records():
    """The multi-rank record transport (counts, then records in source-rank
    order) on world_size 2 with gloo."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_xchg_main, args=(2, port, result), nprocs=2, join=True)
    for dst in range(2):
        n, rows = result[dst]
        expect = [[src, dst, k] for src in range(2) for k in range((src + dst) % 3 + 1)]
        assert n == len(expect) and rows == expect


def _seg_main(rank, world, port, result):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rec, seg = 64, 8
    send = torch.zeros((world, seg, rec), dtype=torch.uint8)
    scnt = torch.tensor([(rank + 2 * d) % 5 + 1 for d in range(world)], dtype=torch.int32)
    for d in range(world):
        for k in range(int(scnt[d])):
            send[d, k, :3] = torch.tensor([rank, d, k], dtype=torch.uint8)
    recv = torch.full((world * seg + 5, rec), 255, dtype=torch.uint8)   # receive capacity > nranks x seg
    rcnt = torch.zeros(world, dtype=torch.int32)
    M.exchange_segments(send.reshape(-1, rec), scnt, recv, rcnt, world, dist)
    uniform = (rcnt.tolist(), recv[: world * seg, :3].tolist(), recv[world * seg:, 0].tolist())
    # per-peer segments: rank r sends caps[r][d] records to d (back to back), d receives them
    # back to back in source order
    caps = [[6, 3], [2, 7]]
    sc, rc = caps[rank], [caps[0][rank], caps[1][rank]]
    flat = torch.zeros((sum(sc), rec), dtype=torch.uint8)
    off = 0
    for d in range(world):
        for k in range(min(int(scnt[d]), sc[d])):
            flat[off + k, :3] = torch.tensor([rank, d, k], dtype=torch.uint8)
        off += sc[d]
    recv2 = torch.full((sum(rc) + 3, rec), 255, dtype=torch.uint8)
    rcnt2 = torch.zeros(world, dtype=torch.int32)
    M.exchange_segments(flat, scnt, recv2, rcnt2, world, dist, sc, rc)
    result[rank] = (uniform, (rcnt2.tolist(), recv2[:, :3].tolist(), rc))
    dist.destroy_process_group()


def test_gloo_exchange_segments():
    """The asynchronous step's transport (fixed segments + device counts, two
    equal-split all-to-alls) on world_size 2 with gloo: segment r of rank d's
    receive buffer is rank r's send segment d, counts alongside, the rest of the
    receive buffer untouched."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_seg_main, args=(2, port, result), nprocs=2, join=True)
    for dst in range(2):
        (rcnt, rows, tail), (rcnt2, rows2, rc) = result[dst]
        assert rcnt == [(src + 2 * dst) % 5 + 1 for src in range(2)]
        for src in range(2):
            for k in range(rcnt[src]):
                assert rows[8 * src + k] == [src, dst, k]
        assert tail == [255] * 5
        assert rcnt2 == rcnt
        off = 0
        for src in range(2):
            for k in range(min(rcnt2[src], rc[src])):
                assert rows2[off + k] == [src, dst, k]
            off += rc[src]
        assert rows2[off:] == [[255, 255, 255]] * 3


def test_droplet_kd_beats_static_split():
    """Heterogeneous workload (off-centre droplet; the
    direction of Fig. 7): the cost-weighted k-d tree balances the
    Eq. 6 load far better than equal-volume boxes."""
    s = S.droplet(L=50.0, R=13.0)                # 20 cells per axis
    cost = M.global_costs(s)
    nz, ny, nx = cost.shape
    for p in (2, 4, 8):
        boxes, loads = M.kd_decompose(cost, p)
        assert loads.sum() == pytest.approx(cost.sum())
        kd = loads.max() / loads.mean()
        # static: equal slabs along x (p = 2), then also y (4), then z (8)
        cuts = [[0, nx // 2, nx], [0, ny // 2, ny] if p >= 4 else [0, ny], [0, nz // 2, nz] if p >= 8 else [0, nz]]
        st = [cost[z0:z1, y0:y1, x0:x1].sum()
              for x0, x1 in zip(cuts[0], cuts[0][1:]) for y0, y1 in zip(cuts[1], cuts[1][1:])
              for z0, z1 in zip(cuts[2], cuts[2][1:])]
        static = max(st) / np.mean(st)
        assert kd < 1.25 and static > 1.5 * kd, (p, kd, static)


def _puts_main(rank, world, port, result):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rb = 64
    caps = [[6, 3, 5], [2, 7, 4], [9, 1, 8]]                 # caps[src][dst]: per-peer segments
    recv_caps = [caps[s][rank] for s in range(world)]
    bases = [(d + 1) << 40 for d in range(world)]            # each rank's symmetric allocation
    recv_off, cnt_off = 4096 * (rank + 1), 256 * (rank + 3)  # layouts may differ per rank
    mine = [recv_off, cnt_off] + [sum(recv_caps[:s]) for s in range(world)]
    t = torch.tensor(mine, dtype=torch.int64)
    allt = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(allt, t)
    rec, cnt = M.peer_target_addrs(rank, bases, [x.tolist() for x in allt], rb)
    got = [torch.empty(2 * world, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(got, torch.tensor(rec + cnt, dtype=torch.int64))
    # where every source's records and count land in this rank's buffers
    result[rank] = (mine, [g.tolist() for g in got])
    dist.destroy_process_group()


def test_gloo_direct_put_targets():
    """Direct puts across ranks (DecomposedRun(direct=True) over NCCL, peer pointers of
    symmetric memory): the addresses rank src stores to for rank d -- its base plus d's
    receive-buffer offset plus d's segment offset for src, and d's count entry src -- are
    exactly where d's import reads source src (world_size 3, gloo, per-peer segments,
    different layouts per rank)."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_puts_main, args=(3, port, result), nprocs=3, join=True)
    caps = [[6, 3, 5], [2, 7, 4], [9, 1, 8]]
    for d in range(3):
        mine, got = result[d]
        base = (d + 1) << 40
        assert mine[0] == 4096 * (d + 1) and mine[1] == 256 * (d + 3)
        for src in range(3):
            seg_off = sum(caps[s][d] for s in range(src))
            assert got[src][d] == base + mine[0] + 64 * seg_off
            assert got[src][3 + d] == base + mine[1] + 4 * src
