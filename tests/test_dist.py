"""Multi-rank plumbing of bench.py on CPU (gloo, world size 2).

Config 5 shards independent systems across ranks with no data-path
collective: rank r owns systems [r*S, (r+1)*S).  These tests
check that the per-rank inputs are exactly the slices of the single-process
batch (so N ranks together solve the same systems as one rank with N*S), and
that the timing reduction is the max over ranks.
"""
import os
import socket
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, S, size, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port),
                       "WORLD_SIZE": str(world), "RANK": str(rank), "LOCAL_RANK": str(rank)})
    import bench
    D = bench.Dist()
    try:
        M, vals, vin = bench.make_inputs(5, size, S, D.rank * S)
        t = D.max(float(rank + 1) * 1.5)
        D.barrier()
        q.put((rank, vals, vin, t, D.world))
    finally:
        D.close()


def test_config5_sharding_gloo_world2():
    world, S, size = 2, 2, 6
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, size, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, vals, vin, t, w = q.get(timeout=180)
        got[rank] = (vals, vin, t, w)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import bench
    M, vals_all, vin_all = bench.make_inputs(5, size, world * S, 0)
    nnz, n = M.nnz, M.n
    for r in range(world):
        vals, vin, t, w = got[r]
        assert w == world
        assert t == 1.5 * world  # max over ranks
        assert np.array_equal(vals, vals_all[r * S * nnz:(r + 1) * S * nnz])
        assert np.array_equal(vin, vin_all[r * S * n:(r + 1) * S * n])
    # the two ranks own different systems
    assert not np.array_equal(got[0][0], got[1][0])


# ---------------------------------------------------------------------------
# config 1: rank 0 solves, x slices go point-to-point, y rows shard
# ---------------------------------------------------------------------------
def _rows_spmv(rowptr, colidx, vals_csr, r0, r1, x):
    """Sequential ascending-column row sums (the order sfg_spmv_rows uses)."""
    y = np.zeros(r1 - r0)
    for r in range(r0, r1):
        acc = 0.0
        for p in range(rowptr[r], rowptr[r + 1]):
            acc = acc + vals_csr[p] * x[colidx[p]]
        y[r - r0] = acc
    return y


def _shard_worker(rank, world, port, k, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port),
                       "WORLD_SIZE": str(world), "RANK": str(rank), "LOCAL_RANK": str(rank)})
    import torch
    import bench
    from paper_2111_12238_b200 import shard
    D = bench.Dist()
    try:
        M = _laplacian2d(k)
        rowptr, colidx = shard.csr_pattern(M[1], M[2], M[0])
        vcsr = _csr_values(M, rowptr)
        x_full = np.random.default_rng(3).standard_normal(M[0])
        seen = {}

        def solve():
            return torch.from_numpy(x_full.copy())

        def spmv(r0, r1, x, y):
            xs = x.numpy()
            lo, hi = S.ranges[rank]
            seen["x"] = xs[lo:hi].copy()
            y[:r1 - r0] = torch.from_numpy(_rows_spmv(rowptr, colidx, vcsr, r0, r1, xs))

        S = shard.ShardedSpmv(D.td, D.rank, D.world, M[0], rowptr, colidx, torch.device("cpu"),
                              solve=solve, spmv=spmv)
        y = S.step().numpy().copy()
        q.put((rank, y, seen.get("x"), S.ranges[rank], S.shards[rank]))
    finally:
        D.close()


def _laplacian2d(k):
    """5-point 2-D Laplacian k^2 in natural order, as (n, colptr, rowidx, values)."""
    n = k * k
    cols = [[] for _ in range(n)]
    for j in range(n):
        r, c = divmod(j, k)
        ent = []
        if r > 0:
            ent.append((j - k, -1.0))
        if c > 0:
            ent.append((j - 1, -1.0))
        ent.append((j, 4.0 + 0.01 * j))
        if c < k - 1:
            ent.append((j + 1, -1.0 - 1e-3 * j))
        if r < k - 1:
            ent.append((j + k, -1.0))
        cols[j] = ent
    colptr = np.zeros(n + 1, dtype=np.int64)
    colptr[1:] = np.cumsum([len(e) for e in cols])
    rowidx = np.array([i for e in cols for i, _ in e], dtype=np.int64)
    vals = np.array([v for e in cols for _, v in e])
    return n, colptr, rowidx, vals


def _csr_values(M, rowptr):
    n, colptr, rowidx, vals = M
    order = np.argsort(rowidx, kind="stable")
    return vals[order]


def test_row_shards_and_halo():
    from paper_2111_12238_b200 import shard
    k = 16
    M = _laplacian2d(k)
    rowptr, colidx = shard.csr_pattern(M[1], M[2], M[0])
    assert shard.row_shards(10, 3) == [(0, 4), (4, 8), (8, 10)]
    assert shard.row_shards(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    sh = shard.row_shards(M[0], 4)
    rg = shard.x_ranges(rowptr, colidx, sh)
    # natural order: each interior boundary reads one grid row (k entries) across it
    assert shard.halo_rows(sh, rg) == [k, 2 * k, 2 * k, k]
    assert shard.x_ranges(rowptr, colidx, [(5, 5)]) == [(5, 5)]
    # ascending columns within each row
    for r in range(M[0]):
        seg = colidx[rowptr[r]:rowptr[r + 1]]
        assert np.all(np.diff(seg) > 0)


def _run_shards(world, k):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, y, xs, rng, sh = q.get(timeout=180)
        got[rank] = (y, xs, rng, sh)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


def test_config1_row_sharded_spmv_gloo():
    """world 2 and a ragged world 3: every rank ends with the y a single
    process computes, bit for bit, and non-zero ranks received exactly the x
    slice their rows read."""
    from paper_2111_12238_b200 import shard
    k = 13  # n = 169: ragged across 3 ranks
    M = _laplacian2d(k)
    rowptr, colidx = shard.csr_pattern(M[1], M[2], M[0])
    vcsr = _csr_values(M, rowptr)
    x_full = np.random.default_rng(3).standard_normal(M[0])
    y_ref = _rows_spmv(rowptr, colidx, vcsr, 0, M[0], x_full)
    for world in (2, 3):
        got = _run_shards(world, k)
        for r in range(world):
            y, xs, (lo, hi), _ = got[r]
            assert np.array_equal(y, y_ref)
            assert np.array_equal(xs, x_full[lo:hi])
