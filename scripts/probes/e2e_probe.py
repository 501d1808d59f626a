"""e2e probe: host-buffer multiply through the C-ABI with pinned vs pageable
buffers, against the device-resident multiply (cfg2 and cfg5)."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2106_04487_b200 as fkt  # noqa: E402

for cfg in (2, 5):
    c = bench.CONFIGS[cfg]
    x, w = fkt.synthConfig(cfg, c["n"])
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(c["kernel"], c["params"]),
                  fkt.FktOptions(p=c["p"], theta=c["theta"], leafCapacity=c["leaf"]))
    nrhs = c["nrhs"]
    W = np.asfortranarray(w.reshape(c["n"], nrhs)) if nrhs > 1 else w
    yd = torch.from_numpy(np.ascontiguousarray(W.T if nrhs > 1 else W)).cuda()
    zd = torch.empty_like(yd)
    st = torch.cuda.Stream()
    for _ in range(3):
        pl.multiply_device(yd, zd, stream=st)
    st.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        pl.multiply_device(yd, zd, stream=st)
    st.synchronize()
    dev = (time.perf_counter() - t0) / 10
    yp = torch.from_numpy(np.ascontiguousarray(W.T if nrhs > 1 else W)).pin_memory()
    zp = torch.empty_like(yp).pin_memory()
    ya = np.ascontiguousarray(W.T if nrhs > 1 else W).copy()
    za = np.empty_like(ya)

    def run(yy, zz, k=8):
        for _ in range(2):
            fkt._check(fkt.lib.fkt_plan_multiply(pl._h, C.cast(C.c_void_p(yy), C.POINTER(C.c_double)),
                                                 C.cast(C.c_void_p(zz), C.POINTER(C.c_double)), nrhs))
        t0 = time.perf_counter()
        for _ in range(k):
            fkt._check(fkt.lib.fkt_plan_multiply(pl._h, C.cast(C.c_void_p(yy), C.POINTER(C.c_double)),
                                                 C.cast(C.c_void_p(zz), C.POINTER(C.c_double)), nrhs))
        return (time.perf_counter() - t0) / k

    pin = run(yp.data_ptr(), zp.data_ptr())
    pag = run(ya.ctypes.data, za.ctypes.data)
    mb = yd.numel() * 8 / 1e6
    print(f"cfg{cfg}: device {dev*1e3:.2f} ms, pinned e2e {pin*1e3:.2f} ms, pageable e2e {pag*1e3:.2f} ms "
          f"({mb:.0f} MB each way)", flush=True)
    del pl
    torch.cuda.empty_cache()
