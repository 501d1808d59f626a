"""TEST INFRASTRUCTURE ONLY — ctypes access to the reference build.

Loads oracle/_ref/libfktref.so: the UNMODIFIED reference sources
(/root/reference/proj/src, compiled by oracle/Makefile) plus the driver
oracle/ref_driver.cpp. Only tests/, __graft_entry__.smoke() and bench.py's
reference / cpu_baseline legs may import this module. It is the checker,
never the thing measured for the product.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libfktref.so")

_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{REF_SO} missing: run `make -C {HERE} ref` where /root/reference exists")
        L = C.CDLL(REF_SO)
        d, u32, i32, ll, u64 = (C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.POINTER(C.c_int),
                                C.POINTER(C.c_longlong), C.POINTER(C.c_uint64))
        sigs = {
            "fktref_last_error": (C.c_char_p,),
            "fktref_config_dims": (C.c_int, C.c_int, i32, i32),
            "fktref_gen_config": (C.c_int, C.c_int, C.c_int, C.c_uint64, d, d),
            "fktref_gen_cloud": (C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_uint64, d, d),
            "fktref_plan_create": (C.c_void_p, C.c_int, C.c_int, d, C.c_char_p, C.c_char_p, C.c_int, C.c_double,
                                   C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double),
            "fktref_plan_destroy": (None, C.c_void_p),
            "fktref_plan_seconds": (C.c_double, C.c_void_p),
            "fktref_plan_info": (C.c_int, C.c_void_p, ll, ll, ll, i32, ll),
            "fktref_plan_tree": (C.c_int, C.c_void_p, u32, u32, u32, i32, i32, d, d, d, d, ll, u32, ll, u32, d),
            "fktref_plan_multiply": (C.c_int, C.c_void_p, d, d, C.c_int),
            "fktref_dense": (C.c_int, C.c_int, C.c_int, d, C.c_char_p, C.c_char_p, d, d, C.c_int, C.c_int,
                             C.c_double),
            "fktref_dense_rows": (C.c_int, C.c_int, C.c_int, d, C.c_char_p, C.c_char_p, d, C.c_int,
                                  C.POINTER(C.c_int64), d, C.c_int, C.c_int, C.c_double),
            "fktref_fingerprints": (C.c_int, C.c_void_p, u64, u64, u64),
            "fktref_tbar": (C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, d, C.c_char_p, C.c_int),
            "fktref_compression_ranks": (C.c_int, C.c_char_p, C.c_char_p, C.c_int, C.c_int, i32),
            "fktref_addition_normalizer": (C.c_double, C.c_int, C.c_int),
            "fktref_harmonics": (C.c_int, C.c_int, C.c_int, d, d),
            "fktref_kernel_jet": (C.c_int, C.c_char_p, C.c_char_p, C.c_double, C.c_int, d),
            "fktref_tbar_serialize": (C.c_longlong, C.c_int, C.c_int, C.c_char_p, C.c_longlong),
            "fktref_tbar_deserialize": (C.c_int, C.c_char_p),
            "fktref_cg_solve": (C.c_int, C.c_int, C.c_int, d, C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_double,
                                C.c_int, C.c_int, C.c_double, d, d, C.c_double, C.c_int, C.c_int, d, i32, d, i32,
                                i32),
            "fktref_gp_posterior_mean": (C.c_int, C.c_int, C.c_int, d, d, d, C.c_char_p, C.c_char_p, C.c_int, d,
                                         C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                         C.c_int, C.c_int, C.c_int, C.c_double, d, i32, d, i32, i32),
        }
        for name, (res, *args) in sigs.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _kv(params: Optional[Dict[str, float]]) -> bytes:
    return ",".join(f"{k}={float(v)!r}" for k, v in (params or {}).items()).encode()


def gen_config(cfg: int, n: int, seed: int = 42):
    L = lib()
    dd, rr = C.c_int(), C.c_int()
    L.fktref_config_dims(cfg, C.byref(dd), C.byref(rr))
    x = np.empty((n, dd.value))
    w = np.empty((rr.value, n))
    if L.fktref_gen_config(cfg, n, seed, _dp(x), _dp(w)) != 0:
        raise RuntimeError(L.fktref_last_error().decode())
    return x, (w[0] if rr.value == 1 else w.T)


def gen_cloud(kind: str, n: int, d: int, seed: int):
    L = lib()
    x = np.empty((n, d))
    y = np.empty(n)
    if L.fktref_gen_cloud(kind.encode(), n, d, seed, _dp(x), _dp(y)) != 0:
        raise RuntimeError(L.fktref_last_error().decode())
    return x, y


class RefPlan:
    """The reference fkt::FktPlan (transform.cpp:39-204), CPU."""

    def __init__(self, x, kernel: str, params=None, p=4, theta=0.75, leaf=512, compression=0, eager=False,
                 threads=0, diagonal=None, barnes_hut=False):
        L = lib()
        if barnes_hut:
            compression = -1  # ref_driver.cpp: FktOptions::barnesHut
        self.x = np.ascontiguousarray(x, dtype=np.float64)
        self.n, self.d = self.x.shape
        self.h = L.fktref_plan_create(self.n, self.d, _dp(self.x), kernel.encode(), _kv(params), p, theta, leaf,
                                      compression, int(eager), threads, int(diagonal is not None),
                                      float(diagonal or 0.0))
        if not self.h:
            raise RuntimeError(L.fktref_last_error().decode())
        nodes, ft, nt, cc = C.c_longlong(), C.c_longlong(), C.c_longlong(), C.c_longlong()
        comp = C.c_int()
        L.fktref_plan_info(self.h, C.byref(nodes), C.byref(ft), C.byref(nt), C.byref(comp), C.byref(cc))
        self.nodes, self.far_total, self.near_total = nodes.value, ft.value, nt.value
        self.compressed, self.coef = bool(comp.value), cc.value
        self.plan_seconds = L.fktref_plan_seconds(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().fktref_plan_destroy(self.h)
            self.h = None

    def multiply(self, y):
        y = np.asfortranarray(np.asarray(y, dtype=np.float64))
        nrhs = 1 if y.ndim == 1 else y.shape[1]
        z = np.empty_like(y, order="F")
        if lib().fktref_plan_multiply(self.h, _dp(y), _dp(z), nrhs) != 0:
            raise RuntimeError(lib().fktref_last_error().decode())
        return z

    def tree(self):
        """dict of reference tree arrays (pre-order) and sets (original indices)."""
        n, d, nn = self.n, self.d, self.nodes
        u32 = lambda k: np.empty(k, np.uint32)
        t = dict(order=u32(n), begin=u32(nn), end=u32(nn), left=np.empty(nn, np.int32),
                 right=np.empty(nn, np.int32), radius=np.empty(nn), center=np.empty((nn, d)),
                 boxLo=np.empty((nn, d)), boxHi=np.empty((nn, d)), farOff=np.empty(nn + 1, np.int64),
                 far=u32(max(1, self.far_total)), nearOff=np.empty(nn + 1, np.int64),
                 near=u32(max(1, self.near_total)), perm=np.empty((n, d)))
        P = lambda a, T: a.ctypes.data_as(C.POINTER(T))
        lib().fktref_plan_tree(self.h, P(t["order"], C.c_uint32), P(t["begin"], C.c_uint32),
                               P(t["end"], C.c_uint32), P(t["left"], C.c_int), P(t["right"], C.c_int),
                               _dp(t["radius"]), _dp(t["center"]), _dp(t["boxLo"]), _dp(t["boxHi"]),
                               P(t["farOff"], C.c_longlong), P(t["far"], C.c_uint32),
                               P(t["nearOff"], C.c_longlong), P(t["near"], C.c_uint32), _dp(t["perm"]))
        t["far"] = t["far"][: self.far_total]
        t["near"] = t["near"][: self.near_total]
        return t

    def fingerprints(self):
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        lib().fktref_fingerprints(self.h, C.byref(a), C.byref(b), C.byref(c))
        return f"{a.value:016x}", f"{b.value:016x}", f"{c.value:016x}"


def dense(x, kernel, params, y, threads=0, diagonal=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    z = np.empty(x.shape[0])
    L = lib()
    if L.fktref_dense(x.shape[0], x.shape[1], _dp(x), kernel.encode(), _kv(params), _dp(y), _dp(z), threads,
                      int(diagonal is not None), float(diagonal or 0.0)) != 0:
        raise RuntimeError(L.fktref_last_error().decode())
    return z


def dense_rows(x, kernel, params, y, rows, threads=0, diagonal=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    z = np.empty(r.size)
    L = lib()
    if L.fktref_dense_rows(x.shape[0], x.shape[1], _dp(x), kernel.encode(), _kv(params), _dp(y), r.size,
                           r.ctypes.data_as(C.POINTER(C.c_int64)), _dp(z), threads, int(diagonal is not None),
                           float(diagonal or 0.0)) != 0:
        raise RuntimeError(L.fktref_last_error().decode())
    return z


def tbar(d, p, k, j, m):
    """(tbarDouble, 'num/den') from the reference's CoefficientTable."""
    v = C.c_double()
    buf = C.create_string_buffer(4096)
    if lib().fktref_tbar(d, p, k, j, m, C.byref(v), buf, 4096) != 0:
        raise RuntimeError(lib().fktref_last_error().decode())
    return v.value, buf.value.decode()


def compression_ranks(kernel, params, d, p):
    ranks = (C.c_int * (p + 1))()
    if lib().fktref_compression_ranks(kernel.encode(), _kv(params), d, p, ranks) != 0:
        raise RuntimeError(lib().fktref_last_error().decode())
    return list(ranks)


def addition_normalizer(d, k):
    return lib().fktref_addition_normalizer(d, k)


def harmonics(d, p, point):
    pt = np.ascontiguousarray(point, dtype=np.float64)
    out = np.empty(4096)
    cnt = lib().fktref_harmonics(d, p, _dp(pt), _dp(out))
    if cnt < 0:
        raise RuntimeError(lib().fktref_last_error().decode())
    return out[:cnt]


def kernel_jet(kernel, params, r, order):
    out = np.empty(order + 1)
    if lib().fktref_kernel_jet(kernel.encode(), _kv(params), r, order, _dp(out)) != 0:
        raise RuntimeError(lib().fktref_last_error().decode())
    return out


def fingerprint_arrays(order, far_off, far, near_off, near, radius, center):
    """SURVEY Appendix A fingerprints from arrays (FNV-1a folds)."""
    P = 1099511628211
    M = (1 << 64) - 1
    h = 1469598103934665603
    for v in order.tolist():
        h = ((h ^ v) * P) & M
    ho = h
    h = 1469598103934665603
    g = 1469598103934665603
    nodes = len(far_off) - 1
    rb = radius.view(np.uint64)
    cb = np.ascontiguousarray(center).view(np.uint64)
    for b in range(nodes):
        for v in far[far_off[b]:far_off[b + 1]].tolist():
            h = ((h ^ ((v + b * 0x9E3779B97F4A7C15) & M)) * P) & M
        for v in near[near_off[b]:near_off[b + 1]].tolist():
            h = ((h ^ ((v * 31 + b) & M)) * P) & M
        g = ((g ^ int(rb[b])) * P) & M
        for c in cb[b].tolist():
            g = ((g ^ c) * P) & M
    return f"{ho:016x}", f"{h:016x}", f"{g:016x}"


def _diag(it, res, conv, rs):
    return {"iterations": it.value, "finalResidual": res.value, "converged": bool(conv.value), "restarts": rs.value}


def cg_solve(x, kernel, params, noise, rhs, tol, maxit, jacobi=False, plan=None, diagonal=None):
    """The reference cgSolve (gp.cpp:58-124). plan=None: dense NoisyOperator;
    plan=dict(p=, theta=, leaf=): NoisyOperator over a reference FktPlan.
    kernel "zero" is test_gp.cpp's zero kernel."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    noise = np.ascontiguousarray(noise, dtype=np.float64)
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    out = np.empty(n)
    it, res, conv, rs = C.c_int(), C.c_double(), C.c_int(), C.c_int()
    pl = plan or {}
    if lib().fktref_cg_solve(n, d, _dp(x), kernel.encode(), _kv(params), int(plan is not None), int(pl.get("p", 4)),
                             float(pl.get("theta", 0.75)), int(pl.get("leaf", 512)), int(diagonal is not None),
                             float(diagonal or 0.0), _dp(noise), _dp(rhs), float(tol), int(maxit), int(jacobi),
                             _dp(out), C.byref(it), C.byref(res), C.byref(conv), C.byref(rs)) != 0:
        raise RuntimeError(lib().fktref_last_error().decode())
    return out, _diag(it, res, conv, rs)


def gp_posterior_mean(train, y, noise, kernel, params, test, p=4, theta=0.75, leaf=512, diagonal=None, tol=1e-10,
                      maxit=1000, jacobi=False, dense=False, prior=None):
    """The reference gpPosteriorMean (gp.cpp:126-177)."""
    train = np.ascontiguousarray(train, dtype=np.float64)
    test = np.ascontiguousarray(test, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    noise = np.ascontiguousarray(noise, dtype=np.float64)
    mean = np.empty(test.shape[0])
    it, res, conv, rs = C.c_int(), C.c_double(), C.c_int(), C.c_int()
    if lib().fktref_gp_posterior_mean(train.shape[0], train.shape[1], _dp(train), _dp(y), _dp(noise),
                                      kernel.encode(), _kv(params), test.shape[0], _dp(test), int(p), float(theta),
                                      int(leaf), int(diagonal is not None), float(diagonal or 0.0), float(tol),
                                      int(maxit), int(jacobi), int(dense), int(prior is not None), float(prior or 0.0),
                                      _dp(mean), C.byref(it), C.byref(res), C.byref(conv), C.byref(rs)) != 0:
        raise RuntimeError(lib().fktref_last_error().decode())
    return mean, _diag(it, res, conv, rs)


def tbar_serialize(d: int, p: int) -> str:
    """The reference CoefficientTable::serialize text (coefficients.cpp:113-124)."""
    need = lib().fktref_tbar_serialize(d, p, None, 0)
    if need < 0:
        raise RuntimeError(lib().fktref_last_error().decode())
    buf = C.create_string_buffer(int(need))
    lib().fktref_tbar_serialize(d, p, buf, need)
    return buf.value.decode()


def tbar_deserialize(text: str) -> int:
    """1: parses and equals the computed table; 0: parses, differs; -1: nullopt."""
    return int(lib().fktref_tbar_deserialize(text.encode()))
