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


@pytest.mark.parametrize("cfg", [2, 5])
def test_shards_are_cost_balanced(fkt, cfg):
    """Cuts at any tree position (not only leaf boundaries): the heaviest of 8
    shards carries at most 5% more than the mean of the per-target cost model
    (near evaluations + far pairs x farPairWeight(P) = P // 5)."""
    c = {2: ("matern32", {"sigma": 1.0, "rho": 0.1}, 1000000, 6, 0.5), 5: ("cauchy", {"sigma": 1.0}, 2000000, 6, 0.75)}[cfg]
    x, _ = fkt.synthConfig(cfg, c[2])
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(c[0], c[1]),
                  fkt.FktOptions(p=c[3], theta=c[4], leafCapacity=512))
    t = pl.tree()
    order = t.order().astype(np.int64)
    inv = np.empty_like(order)
    inv[order] = np.arange(order.size)
    sizes = (t.ends.astype(np.int64) - t.begins.astype(np.int64))
    noff, npos = t.nearCsr()
    foff, fpos = t.farCsr()
    cost = np.zeros(order.size, np.int64)
    np.add.at(cost, inv[npos.astype(np.int64)], np.repeat(sizes, np.diff(noff)))
    np.add.at(cost, inv[fpos.astype(np.int64)], max(1, pl.coefficientCount() // 5))
    cum = np.concatenate([[0], np.cumsum(cost)])
    loads = []
    for s in range(8):
        pl.set_shard(s, 8)
        lo, hi = pl.shard_range()
        loads.append(int(cum[hi] - cum[lo]))
    pl.set_shard(0, 1)
    loads = np.array(loads)
    assert loads.max() <= 1.05 * loads.mean(), loads


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_plan_nccl_world1(fkt):
    """ShardedPlan end to end over a real NCCL process group at world size 1:
    the one-call native path (fkt_plan_multiply_sharded: moment all-reduce and
    z broadcasts on the library's own NCCL communicator, one CUDA graph per
    step), 1 and 16 right-hand sides, deterministic mode included."""
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
        assert sp._comm is not None  # the native NCCL path
        st = torch.cuda.Stream()
        z = torch.empty_like(yd)
        for _ in range(3):  # captured once, replayed
            sp.multiply_device(yd, z, stream=st)
        torch.cuda.synchronize()
        assert np.linalg.norm(z.cpu().numpy() - z1) / np.linalg.norm(z1) <= 1e-14
        Y = torch.from_numpy(np.stack([np.roll(y, 3 * r) for r in range(16)])).cuda().contiguous()
        Z1 = pl.multiply_device(Y).cpu().numpy()
        Z = sp.multiply_device(Y, stream=st)
        torch.cuda.synchronize()
        assert np.linalg.norm(Z.cpu().numpy() - Z1) / np.linalg.norm(Z1) <= 1e-14
        sp.close()
        det = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel("matern32", {"sigma": 1.0, "rho": 0.1}),
                       fkt.FktOptions(p=6, theta=0.5, leafCapacity=512, deterministic=True))
        zdet = det.multiply(y)
        sd = ShardedPlan(det)
        zs = sd.multiply_device(yd, stream=st)
        torch.cuda.synchronize()
        assert np.array_equal(zs.cpu().numpy(), zdet)
        sd.close()
    finally:
        dist.destroy_process_group()
