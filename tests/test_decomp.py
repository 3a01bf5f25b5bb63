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


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _rank_main(rank, world, port, result):
    """One rank of the distributed rebalance's host side: the rank bins the molecules it
    owns on the A12 lattice (mardyn_grid_counts, the library's binning), the per-cell
    counts are summed over the ranks (the engine's ncclAllReduce; gloo here), and every
    rank computes Eq. 6 + the k-d tree through the C ABI."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = S.config("c4s")
    mine = np.arange(len(s["r"]))[rank::world]
    counts = M.grid_counts(s["box"], s["rc"], s["r"][mine]).astype(np.int64)
    t = torch.from_numpy(counts)
    dist.all_reduce(t)                                # per-cell counts of all ranks
    cost = M.cell_cost(t.numpy().astype(np.int32))
    boxes, loads = M.kd_decompose(cost, 4)
    gathered = [None] * world
    dist.all_gather_object(gathered, boxes.tolist())
    uid = M.broadcast_unique_id(dist)                 # the NCCL id every rank creates its context with
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    result[rank] = (gathered, int(t.sum()), float(loads.max() / loads.mean()), ids)
    dist.destroy_process_group()


def test_gloo_two_ranks_agree():
    """world_size 2: the reduced per-cell loads give every rank the same k-d tree, equal to
    the partition of the whole system (mardyn_kd_partition), and every rank receives rank
    0's NCCL unique id."""
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_rank_main, args=(2, _free_port(), result), nprocs=2, join=True)
    g0, n0, imb0, ids0 = result[0]
    g1, n1, imb1, ids1 = result[1]
    s = S.config("c4s")
    whole, _ = M.kd_partition(s["box"], s["rc"], s["r"], 4)
    assert g0[0] == g0[1] == g1[0] == g1[1] == whole.tolist()   # every rank builds the same tree
    assert n0 == n1 == len(s["r"])
    assert imb0 == imb1 and imb0 < 1.2
    assert ids0[0] == ids0[1] == ids1[0] and len(ids0[0]) == 128


def test_grid_counts_are_the_oracle_cells(oracle_mod):
    """The library's host binning (used by mardyn_partition and the rebalance) is the
    A12 cell rule: counts equal the oracle's on the same positions."""
    for name in ("c1s", "c2s", "c4s"):
        s = S.config(name)
        o = oracle_mod.System(s)
        _, cnt = o.cells(o.quantize(s["r"]))
        nc = o.ncell
        assert np.array_equal(M.grid_counts(s["box"], s["rc"], s["r"]), cnt.reshape(nc[2], nc[1], nc[0]))


def test_droplet_kd_beats_static_split():
    """Heterogeneous workload (off-centre droplet; the
    direction of Fig. 7): the cost-weighted k-d tree balances the
    Eq. 6 load far better than equal-volume boxes."""
    s = S.droplet(L=50.0, R=13.0)                # 20 cells per axis
    cost = M.cell_cost(M.grid_counts(s["box"], s["rc"], s["r"]))
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
