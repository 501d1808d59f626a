"""GPU: target sharding of the CUDA plan (csrc/shard.cu).

Shards are run one after another on the one GPU (no rank waits on another):
partial moments of every shard are summed, then each shard evaluates its own
targets; the sum of the shard outputs must equal the unsharded MVM, and each
shard's z must vanish outside its owned targets. The torch.distributed
orchestration (ShardedPlan) runs for real with NCCL at world size 1."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("cube", 200000, 3, "matern32", {"sigma": 1.0, "rho": 0.1}, 6, 512, 0.5, 0),
         ("sphere", 150000, 3, "inverse-r", {}, 8, 256, 0.5, 1),
         ("mixture", 100000, 5, "gaussian", {}, 4, 256, 0.75, 1),
         ("mixture", 100000, 2, "cauchy", {"sigma": 1.0}, 6, 512, 0.75, 0),
         ("cube", 60000, 3, "exponential", {}, 5, 128, 0.6, 0)]  # generic (d, p): direct S2M path


def _simulate(fkt, pl, y, shards):
    import torch

    nrhs = 1 if y.dim() == 1 else y.shape[0]
    order = pl.tree().order().astype(np.int64)
    acc = None
    for s in range(shards):
        pl.set_shard(s, shards)
        pl.stage_device(0, y, None, nrhs=nrhs)
        pl.stage_device(1, None, None, nrhs=nrhs)
        m = pl.moments_view(nrhs).clone()
        acc = m if acc is None else acc + m
    total = torch.zeros_like(y)
    ranges = []
    for s in range(shards):
        pl.set_shard(s, shards)
        lo, hi = pl.shard_range()
        ranges.append((lo, hi))
        pl.stage_device(0, y, None, nrhs=nrhs)
        pl.moments_view(nrhs).copy_(acc)
        zs = torch.empty_like(y)
        for st in (2, 3, 4):
            pl.stage_device(st, None, zs if st == 4 else None, nrhs=nrhs)
        torch.cuda.synchronize()
        zh = zs.cpu().numpy().reshape(nrhs, -1)
        owned = np.zeros(zh.shape[1], bool)
        owned[order[lo:hi]] = True
        assert np.all(zh[:, ~owned] == 0.0), "shard wrote outside its targets"
        total += zs
    pl.set_shard(0, 1)
    return total, ranges


@pytest.mark.parametrize("kind,n,d,name,prm,p,leaf,theta,comp", CASES)
def test_sharded_sum_equals_unsharded(fkt, kind, n, d, name, prm, p, leaf, theta, comp):
    import torch

    x, y = fkt.synthCloud(kind, n, d, 17)
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, prm),
                  fkt.FktOptions(p=p, theta=theta, leafCapacity=leaf, compression=fkt.CompressionMode(comp)))
    yd = torch.from_numpy(y).cuda()
    z1 = pl.multiply_device(yd).cpu().numpy()
    for shards in (2, 3, 5):
        z, ranges = _simulate(fkt, pl, yd, shards)
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(shards - 1))
        assert all(hi > lo for lo, hi in ranges)
        err = np.linalg.norm(z.cpu().numpy() - z1) / np.linalg.norm(z1)
        assert err <= 1e-13, (shards, err)
    # unsharded again after set_shard(0, 1): the plain multiply is unchanged
    assert np.linalg.norm(pl.multiply_device(yd).cpu().numpy() - z1) / np.linalg.norm(z1) <= 1e-14


def test_sharded_barnes_hut(fkt):
    import torch

    x, y = fkt.synthCloud("sphere", 100000, 3, 8)
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel("inverse-r"),
                  fkt.FktOptions(theta=0.5, leafCapacity=256, barnesHut=True))
    yd = torch.from_numpy(y).cuda()
    z1 = pl.multiply_device(yd).cpu().numpy()
    z, _ = _simulate(fkt, pl, yd, 3)
    assert np.linalg.norm(z.cpu().numpy() - z1) / np.linalg.norm(z1) <= 1e-13


def test_sharded_multi_rhs(fkt):
    import torch

    x, y = fkt.synthCloud("mixture", 80000, 2, 3)
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel("cauchy", {"sigma": 1.0}),
                  fkt.FktOptions(p=6, theta=0.75, leafCapacity=512))
    Y = torch.from_numpy(np.stack([y, np.roll(y, 5), -2 * y, np.sin(y)])).cuda().contiguous()
    z1 = pl.multiply_device(Y).cpu().numpy()
    z, _ = _simulate(fkt, pl, Y, 4)
    assert np.linalg.norm(z.cpu().numpy() - z1) / np.linalg.norm(z1) <= 1e-13


def test_sharded_sixteen_rhs_tensor_core_paths(fkt):
    # 16 RHS: the RHS-blocked P2M and the FP64 tensor-core M2T under target
    # shards (re-tiled far / P2M lists), 3 shards summed = unsharded
    import torch

    x, y = fkt.synthCloud("mixture", 60000, 2, 4)
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel("cauchy", {"sigma": 1.0}),
                  fkt.FktOptions(p=6, theta=0.75, leafCapacity=512))
    Y = torch.from_numpy(np.stack([np.roll(y, 7 * r) * (1 + 0.1 * r) for r in range(16)])).cuda().contiguous()
    z1 = pl.multiply_device(Y).cpu().numpy()
    z, _ = _simulate(fkt, pl, Y, 3)
    assert np.linalg.norm(z.cpu().numpy() - z1) / np.linalg.norm(z1) <= 1e-13


def test_shards_are_cost_balanced(fkt):
    """Leaf-aligned cuts: the heaviest shard's near+far pair count stays close
    to the mean (the cut rule balances the per-target cost model)."""
    x, _ = fkt.synthConfig(2, 1000000)
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel("matern32", {"sigma": 1.0, "rho": 0.1}),
                  fkt.FktOptions(p=6, theta=0.5, leafCapacity=512))
    t = pl.tree()
    noff, npos = t.nearCsr()
    order = t.order().astype(np.int64)
    inv = np.empty_like(order)
    inv[order] = np.arange(order.size)
    sizes = (t.ends.astype(np.int64) - t.begins.astype(np.int64))
    near_w = np.repeat(sizes, np.diff(noff))
    loads = []
    for s in range(8):
        pl.set_shard(s, 8)
        lo, hi = pl.shard_range()
        tp = inv[npos.astype(np.int64)]
        loads.append(int(near_w[(tp >= lo) & (tp < hi)].sum()))
    pl.set_shard(0, 1)
    loads = np.array(loads)
    assert loads.max() <= 1.15 * loads.mean(), loads


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_plan_nccl_world1(fkt):
    """ShardedPlan end to end over a real NCCL process group (world size 1:
    the exchange is an identity all-reduce, the stage pipeline is the real
    one)."""
    import torch
    import torch.distributed as dist

    from paper_2106_04487_b200.distributed import ShardedPlan

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        x, y = fkt.synthCloud("cube", 100000, 3, 23)
        pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel("matern32", {"sigma": 1.0, "rho": 0.1}),
                      fkt.FktOptions(p=6, theta=0.5, leafCapacity=512))
        yd = torch.from_numpy(y).cuda()
        z1 = pl.multiply_device(yd).cpu().numpy()
        sp = ShardedPlan(pl)
        st = torch.cuda.Stream()
        z = sp.multiply_device(yd, stream=st)
        torch.cuda.synchronize()
        assert np.linalg.norm(z.cpu().numpy() - z1) / np.linalg.norm(z1) <= 1e-14
    finally:
        dist.destroy_process_group()
