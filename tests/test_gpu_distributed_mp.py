"""GPU: the sharded CUDA plan in TWO processes (world size 2, gloo, one GPU).

Each rank builds the real CUDA plan, owns half of the targets (cost-balanced
cuts), computes partial moments from its sources, exchanges them with a gloo
all-reduce (host-staged: no kernel waits on another rank's kernel), evaluates
its own targets and all-reduces z. The summed result must equal the
single-process MVM (reference split: transform.cpp:18-35, 184-204)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, cfg):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2106_04487_b200 as fkt
    from paper_2106_04487_b200.distributed import ShardedPlan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        kind, n, d, name, prm, p, theta, nrhs, det = cfg
        x, y = fkt.synthCloud(kind, n, d, 41)
        pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, prm),
                      fkt.FktOptions(p=p, theta=theta, leafCapacity=256, deterministic=det))
        Y = np.stack([np.roll(y, 11 * r) for r in range(nrhs)]) if nrhs > 1 else y
        sp = ShardedPlan(pl)
        assert sp._comm is None  # gloo: the staged path
        yd = torch.from_numpy(np.ascontiguousarray(Y)).cuda()
        z = sp.multiply_device(yd)
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"z{rank}.npy"), z.cpu().numpy())
        np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array(sp.shard_range()))
    finally:
        dist.destroy_process_group()


CASES = [("cube", 80000, 3, "matern32", {"sigma": 1.0, "rho": 0.1}, 6, 0.5, 1, False),
         ("mixture", 60000, 2, "cauchy", {"sigma": 1.0}, 6, 0.75, 16, False),
         ("sphere", 50000, 3, "inverse-r", {}, 8, 0.5, 1, True)]


@pytest.mark.parametrize("cfg", CASES)
def test_two_process_sharded_cuda_plan(fkt, tmp_path, cfg):
    import torch.multiprocessing as mp

    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path), cfg), nprocs=2, join=True, start_method="spawn")
    z0, z1 = np.load(tmp_path / "z0.npy"), np.load(tmp_path / "z1.npy")
    r0, r1 = np.load(tmp_path / "r0.npy"), np.load(tmp_path / "r1.npy")
    kind, n, d, name, prm, p, theta, nrhs, det = cfg
    assert r0[0] == 0 and r0[1] == r1[0] and r1[1] == n and 0 < r0[1] < n
    np.testing.assert_array_equal(z0, z1)  # every rank ends with all of z
    x, y = fkt.synthCloud(kind, n, d, 41)
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, prm),
                  fkt.FktOptions(p=p, theta=theta, leafCapacity=256, deterministic=det))
    Y = np.stack([np.roll(y, 11 * r) for r in range(nrhs)]) if nrhs > 1 else y
    zr = pl.multiply(np.ascontiguousarray(Y.T) if nrhs > 1 else Y)
    zr = zr.T if nrhs > 1 else zr
    assert np.linalg.norm(z0 - zr) <= 1e-13 * np.linalg.norm(zr)
