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
