"""Multi-GPU FKT MVM: target sharding with one moment exchange.

The reference parallelises one MVM over CPU threads by chunks of nodes, each
thread with its own z, merged in order (transform.cpp:18-35, 184-204). Here
one process per GPU holds the full plan (tree, sets and tables are cheap to
replicate) and owns a contiguous, leaf-aligned, cost-balanced range of tree
positions (fkt_plan_set_shard, csrc/shard.cu). One MVM is then

    stage 0  gather y into tree order              (every rank, all of y)
    stage 1  S2M from the OWNED sources            -> partial node moments
    exchange sum of the moment tables over ranks   (all_reduce, nodes x P x nrhs)
    stage 2  near field of the OWNED targets       (overlaps the exchange)
    stage 3  M2T of the OWNED targets              (after the exchange)
    stage 4  scatter z (owned entries; 0 elsewhere)
    gather   sum of z over ranks                   (optional: every rank gets all of z)

Moments and z are sums of per-rank partials; non-owned z entries are exact
zeros, so the z sum is exact and the only rounding difference from one GPU is
the order of the moment sum (~1e-16 relative).

Transport is torch.distributed: NCCL over NVLink/NVSwitch on B200 ranks (the
moment table is 3 MB at cfg2, tens of microseconds), gloo on CPU for the
host-logic tests. The plan object only needs the stage interface
(set_shard / shard_range / stage_device / moments_view), so the same
orchestration runs against the CUDA plan (FktPlan) and, in the CPU tests, a
dense stand-in with the same interface.
"""
from __future__ import annotations

import contextlib
from typing import Optional


class ShardedPlan:
    """One rank's view of a target-sharded FKT plan.

    plan: an FktPlan (or any object with the stage interface), already built
    on this rank's device from the SAME cloud, kernel and options as on every
    other rank. group: a torch.distributed process group (default: WORLD).
    """

    def __init__(self, plan, group=None):
        import torch.distributed as dist

        self.plan = plan
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        plan.set_shard(self.rank, self.world)
        self._buf = None

    def shard_range(self):
        return self.plan.shard_range()

    def multiply_device(self, y, z=None, stream=None, gather: bool = True):
        """z = K y for this job. y: (n,) or (nrhs, n) tensor on this rank's
        device (CUDA float64 for the GPU plan). With gather=False, z holds only
        the owned targets (zeros elsewhere) and no z exchange is made."""
        import torch
        import torch.distributed as dist

        nrhs = 1 if y.dim() == 1 else int(y.shape[0])
        if z is None:
            z = torch.empty_like(y)
        cuda = y.is_cuda
        st = (stream if stream is not None else torch.cuda.current_stream()) if cuda else None
        ctx = torch.cuda.stream(st) if cuda else contextlib.nullcontext()
        p = self.plan
        p.stage_device(0, y, None, nrhs=nrhs, stream=st)
        p.stage_device(1, None, None, nrhs=nrhs, stream=st)
        work = None
        if self.world > 1:
            mom = p.moments_view(nrhs)
            if self._buf is None or self._buf.numel() != mom.numel() or self._buf.device != mom.device:
                self._buf = torch.empty_like(mom)
            with ctx:
                self._buf.copy_(mom)
                work = dist.all_reduce(self._buf, group=self.group, async_op=True)
        p.stage_device(2, None, None, nrhs=nrhs, stream=st)  # near field overlaps the exchange
        if work is not None:
            with ctx:
                work.wait()
                mom.copy_(self._buf)
        p.stage_device(3, None, None, nrhs=nrhs, stream=st)
        p.stage_device(4, None, z, nrhs=nrhs, stream=st)
        if gather and self.world > 1:
            with ctx:
                dist.all_reduce(z, group=self.group)
        return z


def shard_cuts(leaf_end, leaf_cum_cost, shards: int, n: int):
    """The library's cut rule (fkt_shard_cuts): leaf-aligned cuts balancing the
    cumulative per-leaf cost. Host only."""
    import ctypes as C

    import numpy as np

    from . import _check, lib

    le = np.ascontiguousarray(leaf_end, dtype=np.uint32)
    lc = np.ascontiguousarray(leaf_cum_cost, dtype=np.uint64)
    cuts = np.zeros(shards + 1, dtype=np.uint32)
    _check(lib.fkt_shard_cuts(le.ctypes.data_as(C.POINTER(C.c_uint32)), lc.ctypes.data_as(C.POINTER(C.c_ulonglong)),
                              int(le.size), int(shards), int(n), cuts.ctypes.data_as(C.POINTER(C.c_uint32))))
    return cuts
