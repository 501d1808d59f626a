"""TEST INFRASTRUCTURE ONLY — ctypes front end of the plain-C restatement
(oracle/fkt_oracle.c -> oracle/build/libfkt_oracle.so) with the exact tables
of oracle/tables.py. A CPU checker; never imported by the product.

    t = RestatedTree(x, leaf)           # proj/src/tree.cpp:29-171
    t.sets(theta)                       # proj/src/tree.cpp:173-213
    z = t.multiply(kernel, params, p, y, compression=0)   # transform.cpp:184-204
"""
from __future__ import annotations

import ctypes as C
import math
import os
from typing import Dict, Optional

import numpy as np

from . import tables as T

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "build", "libfkt_oracle.so")

_lib = None

_d = C.POINTER(C.c_double)
_i = C.POINTER(C.c_int)
_u32 = C.POINTER(C.c_uint32)
_ll = C.POINTER(C.c_longlong)


class _Tables(C.Structure):
    _fields_ = [("d", C.c_int), ("p", C.c_int), ("tbar", _d), ("H", C.c_int), ("hdeg", _i), ("chain_m", _i),
                ("chain_phase", _i), ("chain_norm", _d), ("zk", _d), ("compressed", C.c_int), ("ranks", _i),
                ("tgt_off", _i), ("tgt_pow", _i), ("tgt_c", _d), ("src_off", _i), ("src_pow", _i),
                ("src_c", _d)]


def available() -> bool:
    return os.path.exists(SO)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(SO)
        sigs = {
            "fko_tree_build": (C.c_void_p, C.c_int, C.c_int, _d, C.c_int),
            "fko_tree_free": (None, C.c_void_p),
            "fko_tree_node_count": (C.c_int, C.c_void_p),
            "fko_tree_arrays": (None, C.c_void_p, _u32, _u32, _u32, _i, _i, _d, _d, _d, _d, _d),
            "fko_tree_sets": (C.c_int, C.c_void_p, C.c_double, _ll, _ll),
            "fko_tree_set_arrays": (None, C.c_void_p, _ll, _u32, _ll, _u32),
            "fko_fingerprints": (None, C.c_int, _u32, C.c_int, _ll, _u32, _ll, _u32, _d, _d, C.c_int,
                                 C.POINTER(C.c_uint64)),
            "fko_kernel": (C.c_double, C.c_int, _d, C.c_double),
            "fko_kernel_jet": (None, C.c_int, _d, C.c_double, C.c_int, _d),
            "fko_multiply": (C.c_int, C.c_void_p, C.c_int, _d, C.c_double, C.POINTER(_Tables), _d, _d, C.c_int),
            "fko_dense_rows": (C.c_int, C.c_int, C.c_int, _d, C.c_int, _d, C.c_double, _d, C.c_int,
                               C.POINTER(C.c_int64), _d, C.c_int),
        }
        for name, (res, *args) in sigs.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def kernel_params(kernel: str, params: Optional[Dict[str, float]]):
    """(id, [s2, a, is2, rho], value-at-zero) as proj/src/kernels.cpp:37-156."""
    params = params or {}
    sigma = params.get("sigma", 1.0)
    rho = params.get("rho", 1.0)
    kid = T.KERNELS.index(kernel)
    s2 = sigma * sigma
    prm = np.array([s2, math.sqrt(3.0) / rho, 1.0 / (sigma * sigma), rho])
    v0 = {"matern12": s2, "matern32": s2}.get(kernel, 1.0 if kid in (0, 3, 4, 5) else 0.0)
    return kid, prm, v0


def fingerprints(order, far_off, far, near_off, near, radius, center):
    out = (C.c_uint64 * 3)()
    nodes = len(far_off) - 1
    d = center.shape[1]
    order = np.ascontiguousarray(order, np.uint32)
    far_off = np.ascontiguousarray(far_off, np.int64)
    near_off = np.ascontiguousarray(near_off, np.int64)
    far = np.ascontiguousarray(far, np.uint32) if len(far) else np.zeros(1, np.uint32)
    near = np.ascontiguousarray(near, np.uint32) if len(near) else np.zeros(1, np.uint32)
    radius = np.ascontiguousarray(radius, np.float64)
    center = np.ascontiguousarray(center, np.float64)
    lib().fko_fingerprints(len(order), _p(order, C.c_uint32), nodes, _p(far_off, C.c_longlong), _p(far, C.c_uint32),
                           _p(near_off, C.c_longlong), _p(near, C.c_uint32), _p(radius, C.c_double),
                           _p(center, C.c_double), d, out)
    return tuple(f"{v:016x}" for v in out)


class RestatedTree:
    def __init__(self, x, leaf: int):
        self.x = np.ascontiguousarray(x, dtype=np.float64)
        self.n, self.d = self.x.shape
        self.h = lib().fko_tree_build(self.n, self.d, _p(self.x, C.c_double), leaf)
        if not self.h:
            raise ValueError("invalid tree arguments")
        self.nodes = lib().fko_tree_node_count(self.h)
        n, d, nn = self.n, self.d, self.nodes
        self.order = np.empty(n, np.uint32)
        self.begin = np.empty(nn, np.uint32)
        self.end = np.empty(nn, np.uint32)
        self.left = np.empty(nn, np.int32)
        self.right = np.empty(nn, np.int32)
        self.radius = np.empty(nn)
        self.center = np.empty((nn, d))
        self.boxLo = np.empty((nn, d))
        self.boxHi = np.empty((nn, d))
        self.perm = np.empty((n, d))
        lib().fko_tree_arrays(self.h, _p(self.order, C.c_uint32), _p(self.begin, C.c_uint32),
                              _p(self.end, C.c_uint32), _p(self.left, C.c_int), _p(self.right, C.c_int),
                              _p(self.radius, C.c_double), _p(self.center, C.c_double), _p(self.boxLo, C.c_double),
                              _p(self.boxHi, C.c_double), _p(self.perm, C.c_double))
        self.far_off = self.far = self.near_off = self.near = None

    def __del__(self):
        if getattr(self, "h", None):
            lib().fko_tree_free(self.h)
            self.h = None

    def sets(self, theta: float):
        ft, nt = C.c_longlong(), C.c_longlong()
        if lib().fko_tree_sets(self.h, theta, C.byref(ft), C.byref(nt)) != 0:
            raise ValueError("theta must be in (0, 1)")
        self.far_off = np.empty(self.nodes + 1, np.int64)
        self.near_off = np.empty(self.nodes + 1, np.int64)
        self.far = np.empty(max(1, ft.value), np.uint32)
        self.near = np.empty(max(1, nt.value), np.uint32)
        lib().fko_tree_set_arrays(self.h, _p(self.far_off, C.c_longlong), _p(self.far, C.c_uint32),
                                  _p(self.near_off, C.c_longlong), _p(self.near, C.c_uint32))
        self.far = self.far[: ft.value]
        self.near = self.near[: nt.value]
        return self

    def fingerprints(self):
        return fingerprints(self.order, self.far_off, self.far, self.near_off, self.near, self.radius, self.center)

    def multiply(self, kernel: str, params, p: int, y, compression: int = 0, diagonal=None):
        kid, prm, v0 = kernel_params(kernel, params)
        tab = build_tables(kernel, params, self.d, p, compression)
        y = np.ascontiguousarray(y, dtype=np.float64)
        z = np.empty(self.n)
        rc = lib().fko_multiply(self.h, kid, _p(prm, C.c_double), float(v0 if diagonal is None else diagonal),
                                C.byref(tab.struct), _p(y, C.c_double), _p(z, C.c_double), 1)
        if rc != 0:
            raise RuntimeError("fko_multiply failed")
        return z


class _TableHold:
    pass


def build_tables(kernel: str, params, d: int, p: int, compression: int = 0):
    """Assemble fko_tables from the exact restatement (compression: 0 auto, 1 on, 2 off)."""
    W = p + 1
    tb = np.zeros(W * W * W)
    for (k, j, m), q in T.tbar_table(d, p).items():
        tb[(k * W + j) * W + m] = float(q)  # Fraction -> correctly rounded double
    hdeg, cm, ph, nrm = [], [], [], []
    for k in range(p + 1):
        for ch in T.chains(d, k):
            hdeg.append(k)
            mm = [k] + [abs(c) for c in ch] if d > 2 else [k]
            mm = (mm + [0] * (d - 1))[: max(d - 1, 1)]
            cm.extend(mm)
            ph.append(1 if ch[-1] > 0 else (-1 if ch[-1] < 0 else 0))
            nrm.append(T.chain_norm(d, k, ch))
    zk = [T.addition_normalizer(d, k) for k in range(p + 1)]
    rec = T.recurrence(kernel, params)
    compressed = (compression == 0 and rec is not None) or compression == 1
    if compression == 1 and rec is None:
        raise ValueError("no registered derivative recurrence")
    h = _TableHold()
    h.tb = tb
    h.hdeg = np.array(hdeg, np.int32)
    h.cm = np.array(cm, np.int32)
    h.ph = np.array(ph, np.int32)
    h.nrm = np.array(nrm)
    h.zk = np.array(zk)
    ranks, toff, tpow, tc, soff, spow, sc = [], [0], [], [], [0], [], []
    if compressed:
        for rank, tfs, sfs in T.radial_compression(kernel, params, d, p):
            ranks.append(rank)
            for tf, sf in zip(tfs, sfs):
                for pw, c in sorted(tf.items()):
                    tpow.append(pw)
                    tc.append(float(c))
                toff.append(len(tpow))
                for pw, c in sorted(sf.items()):
                    spow.append(pw)
                    sc.append(float(c))
                soff.append(len(spow))
    h.ranks = np.array(ranks or [0], np.int32)
    h.toff, h.tpow, h.tc = np.array(toff, np.int32), np.array(tpow or [0], np.int32), np.array(tc or [0.0])
    h.soff, h.spow, h.sc = np.array(soff, np.int32), np.array(spow or [0], np.int32), np.array(sc or [0.0])
    h.struct = _Tables(d, p, _p(h.tb, C.c_double), len(hdeg), _p(h.hdeg, C.c_int), _p(h.cm, C.c_int),
                       _p(h.ph, C.c_int), _p(h.nrm, C.c_double), _p(h.zk, C.c_double), int(compressed),
                       _p(h.ranks, C.c_int), _p(h.toff, C.c_int), _p(h.tpow, C.c_int), _p(h.tc, C.c_double),
                       _p(h.soff, C.c_int), _p(h.spow, C.c_int), _p(h.sc, C.c_double))
    h.compressed = compressed
    return h


def dense_rows(x, kernel, params, y, rows, diagonal=None):
    kid, prm, v0 = kernel_params(kernel, params)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    z = np.empty(r.size)
    lib().fko_dense_rows(x.shape[0], x.shape[1], _p(x, C.c_double), kid, _p(prm, C.c_double),
                         float(v0 if diagonal is None else diagonal), _p(y, C.c_double), r.size,
                         r.ctypes.data_as(C.POINTER(C.c_int64)), _p(z, C.c_double), 1)
    return z
