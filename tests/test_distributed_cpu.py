"""CPU (gloo, world_size 2): the multi-GPU orchestration of
paper_2106_04487_b200.distributed and the library's shard cut
rule (fkt_shard_cuts, csrc/shard.cu).

The orchestrator only talks to a plan through the stage interface
(set_shard / shard_range / stage_device / moments_view). Here the plan is a
dense stand-in with the FKT structure -- a permutation into tree order, a
near operator, and a far operator factored through node moments
(z = N y + T (S y), the reference's applyNode split, transform.cpp:131-181) --
restricted to the owned targets/sources exactly as the CUDA plan is. The test
checks that two gloo ranks reproduce the unsharded product; the CUDA plan's
own sharding is checked on the GPU (tests/test_gpu_distributed.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class DensePlan:
    """Dense stand-in with the FktPlan stage interface."""

    def __init__(self, n=240, m=17, leaf=20, seed=3):
        rng = np.random.default_rng(seed)
        self.n, self.leaf = n, leaf
        self.order = rng.permutation(n)  # tree position -> original index
        x = rng.uniform(size=(n, 2))[self.order]
        d2 = ((x[:, None, :] - x[None, :, :]) ** 2).sum(-1)
        self.N = np.where(d2 < 0.04, np.exp(-d2), 0.0)  # near operator (positions)
        self.S = rng.standard_normal((m, n))  # moments = S y_pos
        self.T = rng.standard_normal((n, m))  # far = T moments
        self.lo, self.hi = 0, n
        self.mom = None

    def full(self, y):
        yp = y[..., self.order]
        zp = yp @ self.N.T + (yp @ self.S.T) @ self.T.T
        z = np.empty_like(zp)
        z[..., self.order] = zp
        return z

    def set_shard(self, shard, shards):
        from paper_2106_04487_b200.distributed import shard_cuts

        cost = (self.N != 0).sum(1) + 2  # near pairs + a far weight per target
        ends = np.arange(self.leaf, self.n + 1, self.leaf)
        cum = np.cumsum([cost[e - self.leaf:e].sum() for e in ends])
        cuts = shard_cuts(ends, cum, shards, self.n)
        self.lo, self.hi = int(cuts[shard]), int(cuts[shard + 1])

    def shard_range(self):
        return self.lo, self.hi

    def moments_view(self, nrhs=1):
        return self.mom.view(-1)

    def stage_device(self, stage, y=None, z=None, nrhs=1, stream=None):
        lo, hi = self.lo, self.hi
        if stage == 0:
            self.yp = y.numpy()[..., self.order].reshape(nrhs, self.n)
            self.zp = np.zeros((nrhs, self.n))
            self.mom = torch.zeros(nrhs, self.S.shape[0], dtype=torch.float64)
        elif stage == 1:
            self.mom += torch.from_numpy(self.yp[:, lo:hi] @ self.S[:, lo:hi].T)
        elif stage == 2:
            self.zp[:, lo:hi] += self.yp @ self.N[lo:hi].T
        elif stage == 3:
            self.zp[:, lo:hi] += self.mom.numpy() @ self.T[lo:hi].T
        elif stage == 4:
            out = np.empty_like(self.zp)
            out[:, self.order] = self.zp
            z.copy_(torch.from_numpy(out.reshape(z.shape)))


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2106_04487_b200.distributed import ShardedPlan

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        pl = DensePlan()
        sp = ShardedPlan(pl)
        rng = np.random.default_rng(11)
        out = {"range": sp.shard_range()}
        for nrhs in (1, 3):
            y = rng.standard_normal(pl.n) if nrhs == 1 else rng.standard_normal((nrhs, pl.n))
            z = sp.multiply_device(torch.from_numpy(y)).numpy()
            out[f"err{nrhs}"] = float(np.linalg.norm(z - pl.full(y)) / np.linalg.norm(pl.full(y)))
        y = rng.standard_normal(pl.n)
        zp = sp.multiply_device(torch.from_numpy(y), gather=False).numpy()
        owned = np.zeros(pl.n, bool)
        owned[pl.order[pl.lo:pl.hi]] = True
        out["zeros_outside"] = bool(np.all(zp[~owned] == 0.0))
        out["owned_err"] = float(np.abs(zp[owned] - pl.full(y)[owned]).max())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_sharded_multiply_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    import queue
    import time

    t0 = time.time()
    while len(res) < 2 and time.time() - t0 < 300:
        try:
            r, out = q.get(timeout=2)
            res[r] = out
        except queue.Empty:
            assert all(p.exitcode in (None, 0) for p in procs), "a rank died"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (lo0, hi0), (lo1, hi1) = res[0]["range"], res[1]["range"]
    assert lo0 == 0 and hi0 == lo1 and hi1 == 240 and 0 < hi0 < 240
    for r in (0, 1):
        assert res[r]["err1"] <= 1e-14 and res[r]["err3"] <= 1e-14
        assert res[r]["zeros_outside"] and res[r]["owned_err"] <= 1e-12


def test_shard_cuts_leaf_aligned_and_balanced(fkt):
    from paper_2106_04487_b200.distributed import shard_cuts

    rng = np.random.default_rng(5)
    sizes = rng.integers(1, 50, size=300)
    ends = np.cumsum(sizes)
    cost = rng.integers(1, 1000, size=300)
    cum = np.cumsum(cost)
    n = int(ends[-1])
    for shards in (1, 2, 3, 8, 64):
        cuts = shard_cuts(ends, cum, shards, n)
        assert cuts[0] == 0 and cuts[-1] == n and np.all(np.diff(cuts.astype(np.int64)) >= 0)
        assert set(cuts[1:-1].tolist()) <= set(ends.tolist())
        # every shard is within one leaf's cost of the ideal share
        per = [cum[np.searchsorted(ends, c, side="right") - 1] if c > 0 else 0 for c in cuts]
        share = np.diff(per)
        assert np.all(np.abs(share - cum[-1] / shards) <= cost.max())
    # more shards than leaves: empty shards, still a valid cover
    cuts = shard_cuts(ends[:3], cum[:3], 8, int(ends[2]))
    assert cuts[0] == 0 and cuts[-1] == ends[2] and np.all(np.diff(cuts.astype(np.int64)) >= 0)
