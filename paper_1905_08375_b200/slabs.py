"""Slab sharding along axis 0 (the slowest, contiguous axis).

Each rank owns output rows [row_begin, row_end) and reads input rows
[row_begin - halo_lo, row_end + halo_hi). Static per-node fields (delta, C,
kappa) are sliced once at plan creation; u's halo rows are exchanged with the
two neighbours every apply through torch.distributed point-to-point
(NCCL over NVLink on the GPU box, gloo on CPU in the tests). There is no other
collective on the data path: outputs are disjoint.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def slab_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Even split of n axis-0 rows (first n % world ranks get one more)."""
    base, extra = divmod(n, world)
    rb = rank * base + min(rank, extra)
    re = rb + base + (1 if rank < extra else 0)
    return rb, re


@dataclass
class Slab:
    n: int          # rows along axis 0
    stride: int     # nodes per axis-0 row
    halo: int       # rows of halo the operator needs on each side
    rank: int
    world: int

    def __post_init__(self):
        self.row_begin, self.row_end = slab_rows(self.n, self.world, self.rank)
        self.halo_lo = min(self.halo, self.row_begin)
        self.halo_hi = min(self.halo, self.n - self.row_end)
        self.in_begin = self.row_begin - self.halo_lo
        self.in_end = self.row_end + self.halo_hi
        own = self.row_end - self.row_begin
        # slab_rows is deterministic, so every rank checks every interior slab
        # and all ranks raise together (an undersized slab would otherwise
        # leave its neighbours' halos short and block in the exchange)
        for r in range(1, self.world - 1):
            rb, re = slab_rows(self.n, self.world, r)
            if re - rb < self.halo:
                raise ValueError("halo wider than an interior slab; use fewer ranks")
        if own < 1:
            raise ValueError("empty slab")

    @property
    def n_in(self) -> int:
        return (self.in_end - self.in_begin) * self.stride

    @property
    def n_out(self) -> int:
        return (self.row_end - self.row_begin) * self.stride

    def input_slice(self, a: np.ndarray | None):
        """Rows [in_begin, in_end) of a full-grid per-node array."""
        if a is None:
            return None
        return np.ascontiguousarray(a[self.in_begin * self.stride: self.in_end * self.stride])

    def output_slice(self):
        return slice(self.row_begin * self.stride, self.row_end * self.stride)

    def exchange(self, u_in, group=None) -> None:
        """Fill u_in's halo rows from the neighbours' owned rows (in place).

        u_in covers the input rows; its owned part starts at halo_lo rows.
        Each rank sends its first rows down and its last rows up."""
        import torch.distributed as dist
        if self.world == 1:
            return
        s = self.stride
        own0 = self.halo_lo * s
        own1 = own0 + self.n_out
        ops = []
        if self.rank > 0:
            # the lower neighbour's halo_hi is min(halo, n - its row_end) = rows we own
            lower_rb, lower_re = slab_rows(self.n, self.world, self.rank - 1)
            send_rows = min(self.halo, self.n - lower_re)
            ops.append(dist.P2POp(dist.isend, u_in[own0: own0 + send_rows * s].contiguous(),
                                  self.rank - 1, group))
            ops.append(dist.P2POp(dist.irecv, u_in[0: own0], self.rank - 1, group))
        if self.rank < self.world - 1:
            upper_rb, _ = slab_rows(self.n, self.world, self.rank + 1)
            send_rows = min(self.halo, upper_rb)
            ops.append(dist.P2POp(dist.isend, u_in[own1 - send_rows * s: own1].contiguous(),
                                  self.rank + 1, group))
            ops.append(dist.P2POp(dist.irecv, u_in[own1:], self.rank + 1, group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()


def slab_apply(sl: Slab, plan, u_in, out, stream: int = 0) -> None:
    """One sharded fast apply, the sequence bench.py times at N > 1: the part
    of the apply that does not read u's halo rows (plan.apply_fast_dev_begin),
    the halo exchange with the neighbours (NCCL point-to-point; it overlaps
    the begin part on the device), then the rest (plan.apply_fast_dev_end).
    u_in covers the slab's input rows; only its owned rows need to be valid on
    entry."""
    plan.apply_fast_dev_begin(u_in.data_ptr(), out.data_ptr(), stream)
    comps = int(getattr(plan, "components", 1))
    if comps == 1:
        sl.exchange(u_in)
    else:   # vector fields (peridynamics): SoA component planes of n_in nodes, each with its own halos
        for c in range(comps):
            sl.exchange(u_in[c * sl.n_in:(c + 1) * sl.n_in])
    plan.apply_fast_dev_end(u_in.data_ptr(), out.data_ptr(), stream)
