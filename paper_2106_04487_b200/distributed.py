"""Multi-GPU FKT MVM: target sharding with one moment exchange.

The reference parallelises one MVM over CPU threads by chunks of nodes, each
thread with its own z, merged in order (transform.cpp:18-35, 184-204). Here
one process per GPU holds the full plan (tree, sets and tables are cheap to
replicate) and owns a contiguous, cost-balanced range of tree
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

Two transports:

* NCCL process groups with the CUDA plan: the whole MVM is ONE library call
  (fkt_plan_multiply_sharded, csrc/multigpu.cu) on the library's own NCCL
  communicator (its id shared once over the process group): gather, S2M,
  moment all-reduce, near + M2T, a broadcast of every rank's owned z range
  (tree order; no all-reduce of mostly-zero z) and the scatter, captured as
  one CUDA graph, so a step is one graph launch.
* any other group (gloo; CPU tensors or CUDA tensors staged through the
  host): the stage-by-stage orchestration below with torch.distributed
  collectives. The plan object only needs the stage interface (set_shard /
  shard_range / stage_device / moments_view), so it runs against the CUDA
  plan and, in the CPU tests, a dense stand-in with the same interface.
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

    def __init__(self, plan, group=None, native: Optional[bool] = None):
        import torch.distributed as dist

        self.plan = plan
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        plan.set_shard(self.rank, self.world)
        self._buf = None
        self._comm = None
        # the one-call NCCL path: a CUDA plan on an NCCL process group
        if native is None:
            native = dist.get_backend(group) == "nccl" and hasattr(plan, "_h")
        if native:
            self._comm = self._nccl_comm()

    def _nccl_comm(self):
        import ctypes as C

        import torch.distributed as dist

        from . import _check, lib

        idb = C.create_string_buffer(128)
        if self.rank == 0:
            _check(lib.fkt_nccl_unique_id(idb))
        box = [idb.raw if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=self.group)
        comm = C.c_void_p()
        _check(lib.fkt_nccl_comm_create(box[0], self.world, self.rank, C.byref(comm)))
        return comm

    def close(self):
        if self._comm is not None:
            from . import lib

            lib.fkt_nccl_comm_destroy(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

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
        if self._comm is not None and gather:
            import ctypes as C

            from . import _check, lib

            st = stream if stream is not None else torch.cuda.current_stream()
            _check(lib.fkt_plan_multiply_sharded(self.plan._h, C.c_void_p(y.data_ptr()), C.c_void_p(z.data_ptr()), nrhs,
                                                 self._comm, C.c_void_p(st.cuda_stream)))
            return z
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
    """The library's host cut rule (fkt_shard_cuts): cuts at the given boundaries balancing the
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
