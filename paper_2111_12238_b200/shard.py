"""Row-sharded SpMV stage of BASELINE config 1 across ranks.

Config 1 is combo 4, SpTRSV -> SpMV (kernels.hpp:53-68): x = L^{-1} b, then
y = A x.  The solve is one dependent chain, so it stays on rank 0 (north_star:
a dependent solve stays on one GPU).  The SpMV shards by rows with ONE
exchange step:

1. rank 0 runs kernel 1 alone (``sfg_execute_kernel(plan, 1)``);
2. rank 0 sends each rank r the contiguous slice x[lo_r:hi_r] its rows read
   (its own rows plus the halo; +-512 rows for the 2-D 5-point stencil in
   natural order);
3. every rank computes its rows of y with ``sfg_spmv_rows`` -- ascending
   column order, bit-identical with combo 4's kernel 2 (spmv_csc_col,
   kernels.hpp:162-168, accumulates y_r in the same order);
4. the y shards are all-gathered (padded to equal length).

The exchange is written against ``torch.distributed`` tensors so the same
code runs over NCCL (GPU) and gloo (CPU tests, tests/test_dist.py); the
per-rank compute is a callback.
"""
from __future__ import annotations

import numpy as np


def csr_pattern(colptr: np.ndarray, rowidx: np.ndarray, n: int):
    """CSR (rowptr, colidx) of a CSC pattern, ascending columns within each row
    -- the order the plan's CSR of A uses (and spmv_csc_col's per-row order)."""
    colptr = np.asarray(colptr, dtype=np.int64)
    rowidx = np.asarray(rowidx, dtype=np.int64)
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(colptr))
    order = np.argsort(rowidx, kind="stable")
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rowidx, minlength=n), out=rowptr[1:])
    return rowptr, cols[order]


def row_shards(n: int, world: int) -> list[tuple[int, int]]:
    """Equal contiguous row ranges, ceil(n / world) rows each (last may be short)."""
    L = -(-n // world) if world > 0 else 0
    return [(min(r * L, n), min((r + 1) * L, n)) for r in range(world)]


def x_ranges(rowptr: np.ndarray, colidx: np.ndarray,
             shards: list[tuple[int, int]]) -> list[tuple[int, int]]:
    """For each row shard, the contiguous column range [lo, hi) its rows read.
    An empty shard (or one with no nonzeros) reads nothing: (r0, r0)."""
    out = []
    for r0, r1 in shards:
        a, b = int(rowptr[r0]), int(rowptr[r1])
        if b > a:
            seg = colidx[a:b]
            out.append((int(seg.min()), int(seg.max()) + 1))
        else:
            out.append((r0, r0))
    return out


def halo_rows(shards, ranges) -> list[int]:
    """x entries each shard reads from outside its own rows."""
    return [max(0, r0 - lo) + max(0, hi - r1) for (r0, r1), (lo, hi) in zip(shards, ranges)]


class _CudaArray:
    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_tensor(ptr: int, n: int):
    """A float64 torch view of n doubles at a device pointer (no copy) -- e.g.
    the plan's x (``KernelState.device_output(0)``)."""
    import torch
    return torch.as_tensor(_CudaArray(ptr, n), device="cuda")


def plan_callbacks(st, n: int):
    """solve / spmv callbacks over a combo-4 KernelState whose stream is the
    torch current stream (``st.set_stream``)."""
    xptr, _ = st.device_output(0)
    x = device_tensor(xptr, n)

    def solve():
        st.execute_kernel(1, sync=False)
        return x

    def spmv(r0, r1, xv, y):
        st.spmv_rows(r0, r1, xv.data_ptr(), y.data_ptr())

    return solve, spmv


class ShardedSpmv:
    """One step of the sharded config-1 path on one rank.

    ``solve()`` (rank 0 only) runs kernel 1 and returns x as a 1-D float64
    tensor on ``device``; ``spmv(r0, r1, x, y)`` writes y[0:r1-r0] for rows
    [r0, r1) reading x by absolute column.  ``step()`` returns the gathered
    y (length n) on every rank.
    """

    def __init__(self, td, rank: int, world: int, n: int, rowptr, colidx, device,
                 solve=None, spmv=None):
        import torch
        self.td, self.rank, self.world, self.n = td, rank, world, n
        self.torch = torch
        self.shards = row_shards(n, world)
        self.ranges = x_ranges(np.asarray(rowptr), np.asarray(colidx), self.shards)
        self.L = -(-n // world)
        self.solve_fn, self.spmv_fn = solve, spmv
        f64 = torch.float64
        self.xbuf = torch.zeros(n, dtype=f64, device=device) if rank != 0 else None
        self.yshard = torch.zeros(self.L, dtype=f64, device=device)
        self.yall = torch.zeros(self.L * world, dtype=f64, device=device)
        self.nccl = device.type == "cuda"

    def exchange_x(self, x):
        """Rank 0 -> rank r: x[lo_r:hi_r] (point-to-point, one message per rank)."""
        td = self.td
        reqs = []
        if self.rank == 0:
            for r in range(1, self.world):
                lo, hi = self.ranges[r]
                if hi > lo:
                    reqs.append(td.isend(x[lo:hi], dst=r))
        else:
            lo, hi = self.ranges[self.rank]
            if hi > lo:
                reqs.append(td.irecv(self.xbuf[lo:hi], src=0))
        for q in reqs:
            q.wait()
        return x if self.rank == 0 else self.xbuf

    def gather_y(self):
        if self.world == 1:
            return self.yshard[:self.n]
        if self.nccl:
            self.td.all_gather_into_tensor(self.yall, self.yshard)
        else:
            self.td.all_gather(list(self.yall.split(self.L)), self.yshard)
        return self.yall[:self.n]

    def step(self):
        x = self.solve_fn() if self.rank == 0 else None
        xr = self.exchange_x(x) if self.world > 1 else x
        r0, r1 = self.shards[self.rank]
        if r1 > r0:
            self.spmv_fn(r0, r1, xr, self.yshard)
        return self.gather_y()

    def exchanged_bytes(self) -> dict:
        """Bytes moved per step: the x slices (rank 0 out) and the y gather."""
        xs = sum(8 * (hi - lo) for (lo, hi) in self.ranges[1:])
        return {"x_p2p": xs, "y_allgather": 8 * self.L * self.world * (self.world - 1)}
