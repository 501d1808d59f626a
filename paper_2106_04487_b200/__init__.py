"""B200-native Fast Kernel Transform MVM — Python mirror of the reference's
C++ operator API (reference proj/include/fkt/{tree,kernels,transform}.hpp).

Names, argument meaning and error behaviour follow the reference so parity
tests read like its doctest suite:

    cloud = PointCloud.from_array(x)                  # fkt::PointCloud
    k = makeKernel("matern32", {"sigma": 1, "rho": 0.1})
    opts = FktOptions(p=6, theta=0.5, leafCapacity=512)
    p = plan(cloud, k, opts)                          # fkt::plan -> FktPlan
    z = p.multiply(y)                                 # FktPlan::multiply
    p.tree().node(0).farSet                           # PartitionTree view

Everything computes on the GPU through the C-ABI (include/fkt_cuda.h); there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Dict, Optional, Sequence

import numpy as np

from . import _lib as _L

lib = _L.lib

__all__ = [
    "PointCloud", "IsotropicKernel", "makeKernel", "builtinKernelNames", "CompressionMode", "FktOptions",
    "TreeNode", "PartitionTree", "FktPlan", "plan", "denseMultiply", "denseRows", "relativeError",
    "expansionSize", "FktError", "DimensionMismatchError", "ZeroReferenceError", "OrderTooLargeError",
    "NotRecurrenceKernelError", "SingularAtZeroError", "UnsupportedOnGpuError", "CudaError",
    "synthCloud", "synthConfig", "configDims", "tbar", "compressionRanks", "additionNormalizer",
]


# --- errors (reference exception types) ------------------------------------
class FktError(Exception):
    pass


class InvalidArgument(FktError, ValueError):
    """std::invalid_argument"""


class DimensionMismatchError(InvalidArgument):
    """fkt::DimensionMismatchError (transform.hpp:17-20)"""


class ZeroReferenceError(InvalidArgument):
    """fkt::ZeroReferenceError (transform.hpp:22-25)"""


class OrderTooLargeError(InvalidArgument):
    """fkt::OrderTooLargeError (coefficients.hpp:23-28)"""


class NotRecurrenceKernelError(InvalidArgument):
    """fkt::NotRecurrenceKernelError (expansion.hpp:27-31)"""


class SingularAtZeroError(FktError, ArithmeticError):
    """fkt::SingularAtZeroError (kernels.hpp:22-26)"""


class UnsupportedOnGpuError(InvalidArgument):
    """A valid reference input this GPU path does not offer (no CPU fallback)."""


class CudaError(FktError, RuntimeError):
    """Device failure."""


_ERRORS = {
    1: InvalidArgument,
    2: DimensionMismatchError,
    3: OrderTooLargeError,
    4: NotRecurrenceKernelError,
    5: SingularAtZeroError,
    6: ZeroReferenceError,
    7: CudaError,
    8: UnsupportedOnGpuError,
    9: FktError,
}


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib.fkt_last_error().decode()
        raise _ERRORS.get(rc, FktError)(msg)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


def _params(params: Dict[str, float]):
    keys = list(params.keys())
    karr = (C.c_char_p * max(1, len(keys)))(*[k.encode() for k in keys])
    varr = (C.c_double * max(1, len(keys)))(*[float(params[k]) for k in keys])
    return karr, varr, len(keys)


# --- point cloud --------------------------------------------------------------
class PointCloud:
    """fkt::PointCloud (tree.hpp:16-28): n points in d dimensions, row-major."""

    def __init__(self, n: int = 0, d: int = 0, x=None):
        self.n = int(n)
        self.d = int(d)
        self.x = np.zeros((self.n, self.d)) if x is None else _f64(x, (self.n, self.d))

    @classmethod
    def from_array(cls, x) -> "PointCloud":
        x = _f64(x)
        if x.ndim != 2:
            raise InvalidArgument("point array must be n x d")
        return cls(x.shape[0], x.shape[1], x)

    def point(self, i: int) -> np.ndarray:
        return self.x[i]


# --- kernels -----------------------------------------------------------------
class IsotropicKernel:
    """A built-in isotropic kernel by name (kernels.hpp:28-78)."""

    def __init__(self, name: str, params: Optional[Dict[str, float]] = None):
        self._name = name
        self._params = dict(params or {})
        rec, hv0, v0 = C.c_int(), C.c_int(), C.c_double()
        k, v, n = _params(self._params)
        _check(lib.fkt_kernel_check(name.encode(), k, v, n, C.byref(rec), C.byref(hv0), C.byref(v0)))
        self._rec = bool(rec.value)
        self._v0 = v0.value if hv0.value else None

    def name(self) -> str:
        return self._name

    def parameters(self) -> Dict[str, float]:
        return dict(self._params)

    def hasDerivativeRecurrence(self) -> bool:
        return self._rec

    def valueAtZero(self) -> Optional[float]:
        return self._v0

    def __call__(self, r, diagonalOverride: Optional[float] = None):
        """K(r); r == 0 uses the override, else the kernel's convention, else raises."""
        rr = _f64(np.atleast_1d(r))
        out = np.empty_like(rr)
        k, v, n = _params(self._params)
        _check(lib.fkt_kernel_eval(self._name.encode(), k, v, n, _dptr(rr), _dptr(out), rr.size,
                                   int(diagonalOverride is not None), float(diagonalOverride or 0.0)))
        return out if np.ndim(r) else float(out[0])

    def evalPositive(self, r):
        return self(r)


def makeKernel(name: str, params: Optional[Dict[str, float]] = None) -> IsotropicKernel:
    """fkt::makeKernel (kernels.cpp:37-156). Unknown names / parameters raise."""
    return IsotropicKernel(name, params)


def builtinKernelNames():
    return [lib.fkt_kernel_name(i).decode() for i in range(lib.fkt_kernel_count())]


# --- options --------------------------------------------------------------------
class CompressionMode(enum.IntEnum):
    Auto = 0
    On = 1
    Off = 2


@dataclass
class FktOptions:
    """fkt::FktOptions (transform.hpp:29-41)."""

    p: int = 4
    theta: float = 0.75
    leafCapacity: int = 512
    compression: CompressionMode = CompressionMode.Auto
    eagerOperators: bool = True
    barnesHut: bool = False
    threads: int = 0
    diagonal: Optional[float] = None
    nearPrecision: int = 64  # additive: 32 selects the FP32 fast near field
    deterministic: bool = False  # additive: bitwise reproducible z (fixed-order sums)

    def _c(self) -> _L.FktOptionsC:
        return _L.FktOptionsC(int(self.p), float(self.theta), int(self.leafCapacity), int(self.compression),
                              int(bool(self.eagerOperators)), int(bool(self.barnesHut)), int(self.threads),
                              int(self.diagonal is not None), float(self.diagonal or 0.0), int(self.nearPrecision),
                              int(bool(self.deterministic)))


# --- tree view -----------------------------------------------------------------
@dataclass
class TreeNode:
    """fkt::TreeNode (tree.hpp:30-41)."""

    boxLo: np.ndarray
    boxHi: np.ndarray
    center: np.ndarray
    radius: float
    begin: int
    end: int
    left: int
    right: int
    farSet: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    nearSet: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))

    def isLeaf(self) -> bool:
        return self.left < 0

    def count(self) -> int:
        return self.end - self.begin


class PartitionTree:
    """fkt::PartitionTree (tree.hpp:43-79), built on the GPU.

    ``PartitionTree(cloud, leafCapacity)`` builds a standalone tree; plans
    expose theirs through ``FktPlan.tree()``.
    """

    def __init__(self, cloud: Optional[PointCloud] = None, leafCapacity: int = 512, *, _handle=None, _dim=None,
                 _owner=None):
        self._owner = _owner  # keeps a plan alive while its borrowed tree view is used
        if _handle is not None:
            self._h = _handle
            self._owned = False
            self._d = int(_dim)
        else:
            h = C.c_void_p()
            _check(lib.fkt_tree_create(cloud.n, cloud.d, _dptr(cloud.x), int(leafCapacity), C.byref(h)))
            self._h = h
            self._owned = True
            self._d = cloud.d
        self._reset()

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "_h", None):
            lib.fkt_tree_destroy(self._h)
            self._h = None

    def _reset(self):
        nodes, depth, ft, nt = C.c_longlong(), C.c_longlong(), C.c_longlong(), C.c_longlong()
        th = C.c_double()
        _check(lib.fkt_tree_sizes(self._h, C.byref(nodes), C.byref(depth), C.byref(ft), C.byref(nt), C.byref(th)))
        self._nodes, self._depth, self._theta = nodes.value, depth.value, th.value
        self._totals = (ft.value, nt.value)
        self._far = self._near = None
        self._order = self._perm = None
        nn, d = self._nodes, self._d
        self.begins = np.empty(nn, np.uint32)
        self.ends = np.empty(nn, np.uint32)
        self.lefts = np.empty(nn, np.int32)
        self.rights = np.empty(nn, np.int32)
        self.radii = np.empty(nn)
        self.centers = np.empty((nn, d))
        self.boxLos = np.empty((nn, d))
        self.boxHis = np.empty((nn, d))
        _check(lib.fkt_tree_nodes(self._h, self.begins.ctypes.data_as(_L._u32), self.ends.ctypes.data_as(_L._u32),
                                  self.lefts.ctypes.data_as(_L._i32), self.rights.ctypes.data_as(_L._i32),
                                  _dptr(self.radii), _dptr(self.centers), _dptr(self.boxLos), _dptr(self.boxHis)))

    # reference accessors
    def nodeCount(self) -> int:
        return self._nodes

    def depth(self) -> int:
        return self._depth

    def theta(self) -> float:
        return self._theta

    def hasInteractionSets(self) -> bool:
        return self._theta > 0.0

    def dimension(self) -> int:
        return self._d

    def pointCount(self) -> int:
        return int(self.ends[0])

    def computeInteractionSets(self, theta: float) -> None:
        _check(lib.fkt_tree_compute_sets(self._h, float(theta)))
        self._reset()

    def order(self) -> np.ndarray:
        if self._order is None:
            order = np.empty(self.pointCount(), np.uint32)
            _check(lib.fkt_tree_order(self._h, order.ctypes.data_as(_L._u32)))
            self._order = order
        return self._order

    def originalIndex(self, pos: int) -> int:
        return int(self.order()[pos])

    def points(self) -> np.ndarray:
        """All permuted coordinates (pointAt for every position), n x d."""
        if self._perm is None:
            perm = np.empty((self.pointCount(), self._d))
            _check(lib.fkt_tree_points(self._h, _dptr(perm)))
            self._perm = perm
        return self._perm

    def pointAt(self, pos: int) -> np.ndarray:
        return self.points()[pos]

    def farCsr(self):
        """(offsets[nodes+1], original indices) of every farSet, ascending per node."""
        if self._far is None:
            self._far = self._sets(lib.fkt_tree_far_sets, self._totals[0])
        return self._far

    def nearCsr(self):
        if self._near is None:
            self._near = self._sets(lib.fkt_tree_near_sets, self._totals[1])
        return self._near

    def _sets(self, fn, total):
        off = np.empty(self._nodes + 1, np.int64)
        idx = np.empty(max(total, 1), np.uint32)
        _check(fn(self._h, off.ctypes.data_as(_L._ll), idx.ctypes.data_as(_L._u32)))
        return off, idx[:total]

    def node(self, i: int) -> TreeNode:
        far = near = np.zeros(0, np.uint32)
        if self.hasInteractionSets():
            fo, fi = self.farCsr()
            no, ni = self.nearCsr()
            far = fi[fo[i]:fo[i + 1]]
            near = ni[no[i]:no[i + 1]]
        return TreeNode(self.boxLos[i].copy(), self.boxHis[i].copy(), self.centers[i].copy(), float(self.radii[i]),
                        int(self.begins[i]), int(self.ends[i]), int(self.lefts[i]), int(self.rights[i]), far, near)


# --- plan ----------------------------------------------------------------------
class FktPlan:
    """fkt::FktPlan (transform.hpp:43-74) on one GPU."""

    def __init__(self, cloud: PointCloud, kernel: IsotropicKernel, options: Optional[FktOptions] = None,
                 _cached: bool = False):
        options = options or FktOptions()
        self._n, self._d = cloud.n, cloud.d
        self._cloud_host, self._cloud_dev = PointCloud(cloud.n, cloud.d, cloud.x.copy()), None
        self._kernel = kernel
        if options.barnesHut:  # transform.cpp:44: a Barnes-Hut plan has p = 0
            import dataclasses

            options = dataclasses.replace(options, p=0)
        self._options = options
        self.d = cloud.d
        h = C.c_void_p()
        k, v, n = _params(kernel.parameters())
        oc = options._c()
        self._cached = _cached
        self.cacheHit = False
        if _cached:
            hit = C.c_int()
            _check(lib.fkt_plan_cache_get(cloud.n, cloud.d, _dptr(self._cloud.x), kernel.name().encode(), k, v, n,
                                          C.byref(oc), C.byref(h), C.byref(hit)))
            self.cacheHit = bool(hit.value)
        else:
            _check(lib.fkt_plan_create(cloud.n, cloud.d, _dptr(self._cloud.x), kernel.name().encode(), k, v, n,
                                       C.byref(oc), C.byref(h)))
        self._h = h
        self._tree = None
        info = _L.FktPlanInfoC()
        _check(lib.fkt_plan_info_get(self._h, C.byref(info)))
        self._info = info

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            if getattr(self, "_cached", False):
                lib.fkt_plan_cache_release(h)
            else:
                lib.fkt_plan_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    def rebuild(self, cloud) -> None:
        """Additive: the same plan on new coordinates of the same n points
        (moving points, e.g. t-SNE iterations). Equals a fresh plan on `cloud`
        with this plan's kernel and options; tree, sets, tiles and moment plan
        are rebuilt on the GPU reusing the plan's buffers (fkt_plan_rebuild)."""
        x = cloud.x if isinstance(cloud, PointCloud) else np.asarray(cloud, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.ndim != 2 or x.shape != (self._n, self._d):
            raise DimensionMismatchError("rebuild: the cloud must have the plan's n points in d dimensions")
        _check(lib.fkt_plan_rebuild(self._h, _dptr(x)))
        # cloud() hands out this array (a view of the caller's when it was
        # already contiguous FP64: no 8nd-byte host copy per re-plan)
        self._cloud_host, self._cloud_dev = PointCloud(self._n, self._d, x), None
        self._after_rebuild()

    def rebuild_device(self, x) -> None:
        """rebuild() with the new coordinates already in device memory: a
        contiguous float64 CUDA tensor of shape (n, d) (fkt_plan_rebuild_device).
        Pending work on torch's current stream is waited for first."""
        import torch

        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()
                and tuple(x.shape) == (self._n, self._d)):
            raise DimensionMismatchError("rebuild_device: need a contiguous float64 CUDA tensor of shape (n, d)")
        torch.cuda.current_stream(x.device).synchronize()
        _check(lib.fkt_plan_rebuild_device(self._h, C.c_void_p(x.data_ptr())))
        self._cloud_host, self._cloud_dev = None, x  # cloud() copies it back on demand
        self._after_rebuild()

    def _after_rebuild(self) -> None:
        self._tree = None
        info = _L.FktPlanInfoC()
        _check(lib.fkt_plan_info_get(self._h, C.byref(info)))
        self._info = info

    @property
    def _cloud(self) -> PointCloud:
        if self._cloud_host is None:
            self._cloud_host = PointCloud(self._n, self._d, self._cloud_dev.cpu().numpy())
        return self._cloud_host

    # reference accessors
    def cloud(self) -> PointCloud:
        return self._cloud

    def kernel(self) -> IsotropicKernel:
        return self._kernel

    def options(self) -> FktOptions:
        return self._options

    def compressed(self) -> bool:
        return bool(self._info.compressed)

    def coefficientCount(self) -> int:
        return int(self._info.coefficient_count)

    def info(self) -> dict:
        return {f: getattr(self._info, f) for f, _ in _L.FktPlanInfoC._fields_}

    PLAN_PHASES = ("tree", "sets", "tables", "tiles", "near_rows", "moments", "other")

    def plan_phases(self) -> dict:
        """Plan-time seconds per phase (fkt_plan_phases)."""
        out = (C.c_double * len(self.PLAN_PHASES))()
        _check(lib.fkt_plan_phases(self._h, out, len(self.PLAN_PHASES)))
        return dict(zip(self.PLAN_PHASES, list(out)))

    def tree(self) -> PartitionTree:
        if self._tree is None:
            th = lib.fkt_plan_tree(self._h)
            self._tree = PartitionTree(_handle=C.c_void_p(th), _dim=self.d, _owner=self)
        return self._tree

    def multiply(self, y) -> np.ndarray:
        """z = K y. y: length n, or n x nrhs (one multiply per column, batched)."""
        y = _f64(y)
        n = self._cloud.n
        if y.ndim == 1:
            if y.shape[0] != n:
                raise DimensionMismatchError("multiply: vector length does not match the point count")
            z = np.empty(n)
            _check(lib.fkt_plan_multiply(self._h, _dptr(y), _dptr(z), 1))
            return z
        if y.ndim != 2 or y.shape[0] != n:
            raise DimensionMismatchError("multiply: vector length does not match the point count")
        yc = np.asfortranarray(y)
        z = np.empty_like(yc, order="F")
        _check(lib.fkt_plan_multiply(self._h, yc.ctypes.data_as(C.POINTER(C.c_double)),
                                     z.ctypes.data_as(C.POINTER(C.c_double)), y.shape[1]))
        return z

    def multiply_device(self, y, z=None, stream=None):
        """Device-resident multiply on torch CUDA tensors (column-major nrhs via shape (nrhs, n))."""
        import torch

        if not (isinstance(y, torch.Tensor) and y.is_cuda and y.dtype == torch.float64 and y.is_contiguous()):
            raise InvalidArgument("multiply_device expects a contiguous float64 CUDA tensor")
        nrhs = 1 if y.dim() == 1 else y.shape[0]
        if y.shape[-1] != self._cloud.n:
            raise DimensionMismatchError("multiply: vector length does not match the point count")
        if z is None:
            z = torch.empty_like(y)
        elif not (isinstance(z, torch.Tensor) and z.is_cuda and z.dtype == torch.float64 and z.is_contiguous()
                  and z.shape == y.shape and z.device == y.device):
            raise InvalidArgument("multiply_device: z must be a contiguous float64 CUDA tensor shaped and placed like y")
        st = stream if stream is not None else torch.cuda.current_stream()
        _check(lib.fkt_plan_multiply_device(self._h, C.c_void_p(y.data_ptr()), C.c_void_p(z.data_ptr()), nrhs,
                                            C.c_void_p(st.cuda_stream)))
        return z

    def stage_device(self, stage: int, y=None, z=None, nrhs: int = 1, stream=None):
        import torch

        st = stream if stream is not None else torch.cuda.current_stream()
        _check(lib.fkt_plan_stage_device(self._h, int(stage), C.c_void_p(y.data_ptr() if y is not None else 0),
                                         C.c_void_p(z.data_ptr() if z is not None else 0), nrhs,
                                         C.c_void_p(st.cuda_stream)))

    def near_forms(self):
        """(Gram-form tiles, all near tiles) of the FP64 near field."""
        g, t = C.c_longlong(), C.c_longlong()
        _check(lib.fkt_plan_near_forms(self._h, C.byref(g), C.byref(t)))
        return int(g.value), int(t.value)

    def kernel_launches(self, nrhs: int = 1) -> int:
        """This library's kernels one multiply launches (memsets excluded)."""
        return int(lib.fkt_plan_kernel_launches(self._h, int(nrhs)))

    # ---- multi-GPU target sharding (see distributed.py) ----------
    def set_shard(self, shard: int, shards: int) -> None:
        """Own the cost-balanced target range `shard` of `shards` (tree positions)."""
        _check(lib.fkt_plan_set_shard(self._h, int(shard), int(shards)))

    def shard_range(self):
        """Owned tree positions [lo, hi)."""
        lo, hi = C.c_longlong(), C.c_longlong()
        _check(lib.fkt_plan_shard_range(self._h, C.byref(lo), C.byref(hi)))
        return int(lo.value), int(hi.value)

    def moments_view(self, nrhs: int = 1):
        """The plan's node-moment table ([rhs][node][P], float64) as a torch CUDA
        tensor sharing its memory (valid until the next reallocation)."""
        import torch

        ptr, per = C.POINTER(C.c_double)(), C.c_longlong()
        _check(lib.fkt_plan_moments_device(self._h, C.byref(ptr), C.byref(per)))
        count = int(per.value) * int(nrhs)

        class _View:
            __cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "version": 3,
                                        "data": (C.cast(ptr, C.c_void_p).value, False), "strides": None}

        return torch.as_tensor(_View(), device="cuda")


def plan(cloud: PointCloud, kernel: IsotropicKernel, options: Optional[FktOptions] = None) -> FktPlan:
    """fkt::plan (transform.cpp:206-208)."""
    return FktPlan(cloud, kernel, options)


def barnesHutMultiply(plan: FktPlan, y) -> np.ndarray:
    """fkt::barnesHutMultiply (transform.cpp:239-243): multiply on a plan built
    with FktOptions(barnesHut=True) (monopole far field about the centres of
    mass, csrc/bh.cu)."""
    if not plan.options().barnesHut:
        raise InvalidArgument("barnesHutMultiply requires a plan built with the Barnes-Hut option")
    return plan.multiply(y)


def cachedPlan(cloud: PointCloud, kernel: IsotropicKernel, options: Optional[FktOptions] = None) -> FktPlan:
    """A plan from the library's plan cache (fkt_plan_cache_get): identical
    (cloud, kernel, options) requests share one device plan; `.cacheHit` says
    whether it was reused. The reference rebuilds plans per call site."""
    return FktPlan(cloud, kernel, options, _cached=True)


def planCacheCapacity(plans: int) -> None:
    _check(lib.fkt_plan_cache_set_capacity(int(plans)))


def planCacheSize() -> int:
    return int(lib.fkt_plan_cache_size())


def denseMultiply(cloud: PointCloud, kernel: IsotropicKernel, y, diagonal: Optional[float] = None,
                  threads: int = 0) -> np.ndarray:
    """fkt::denseMultiply (transform.cpp:210-237), O(N^2) on the GPU."""
    y = _f64(y)
    if y.shape != (cloud.n,):
        raise DimensionMismatchError("denseMultiply: vector length does not match the point count")
    z = np.empty(cloud.n)
    k, v, n = _params(kernel.parameters())
    _check(lib.fkt_dense_multiply(cloud.n, cloud.d, _dptr(cloud.x), kernel.name().encode(), k, v, n, _dptr(y),
                                  _dptr(z), int(diagonal is not None), float(diagonal or 0.0)))
    return z


def denseRows(cloud: PointCloud, kernel: IsotropicKernel, y, rows: Sequence[int],
              diagonal: Optional[float] = None) -> np.ndarray:
    """Rows `rows` of the dense product (validation against sampled rows)."""
    y = _f64(y)
    if y.shape != (cloud.n,):
        raise DimensionMismatchError("denseRows: vector length does not match the point count")
    r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    z = np.empty(r.size)
    k, v, n = _params(kernel.parameters())
    _check(lib.fkt_dense_rows(cloud.n, cloud.d, _dptr(cloud.x), kernel.name().encode(), k, v, n, _dptr(y), r.size,
                              r.ctypes.data_as(_L._i64), _dptr(z), int(diagonal is not None), float(diagonal or 0.0)))
    return z


def relativeError(approx, exact) -> float:
    """fkt::relativeError (transform.cpp:245-255)."""
    a, e = _f64(approx).ravel(), _f64(exact).ravel()
    if a.size != e.size:
        raise DimensionMismatchError("relativeError: length mismatch")
    out = C.c_double()
    _check(lib.fkt_relative_error(_dptr(a), _dptr(e), a.size, C.byref(out)))
    return out.value


# --- Gaussian processes (reference proj/include/fkt/gp.hpp, gp.cpp) -------------
@dataclass
class CgDiagnostics:
    """fkt::CgDiagnostics (gp.hpp:35-40)."""

    iterations: int = 0
    finalResidual: float = 0.0
    converged: bool = False
    restarts: int = 0

    @staticmethod
    def _from(c) -> "CgDiagnostics":
        return CgDiagnostics(int(c.iterations), float(c.final_residual), bool(c.converged), int(c.restarts))


@dataclass
class CgResult:
    """fkt::CgResult (gp.hpp:42-45)."""

    x: np.ndarray
    diagnostics: CgDiagnostics


class NoisyOperator:
    """fkt::NoisyOperator (gp.hpp:17-33, gp.cpp:20-44): y -> K y + noise .* y.

    NoisyOperator(plan, noise) uses the FKT plan; NoisyOperator(cloud, kernel,
    noise, diagonal=None) the dense product (on the GPU)."""

    def __init__(self, a, b, c=None, diagonal: Optional[float] = None):
        if isinstance(a, FktPlan):
            self._plan, self._cloud, self._kernel, self._diag = a, a.cloud(), a.kernel(), a.options().diagonal
            noise = b
        else:
            self._plan, self._cloud, self._kernel, self._diag = None, a, b, diagonal
            noise = c
        self._noise = _f64(noise).ravel()
        if self._noise.size != self._cloud.n:
            raise DimensionMismatchError("NoisyOperator: noise length does not match the point count")
        # gp.cpp:10-16: K(0) under the diagonal convention, 0 when singular
        v0 = self._kernel.valueAtZero()
        self._k0 = float(self._diag) if self._diag is not None else (float(v0) if v0 is not None else 0.0)

    def size(self) -> int:
        return self._cloud.n

    def noise(self) -> np.ndarray:
        return self._noise

    def kernelDiagonal(self) -> float:
        return self._k0

    def apply(self, y) -> np.ndarray:
        y = _f64(y).ravel()
        if y.size != self._cloud.n:
            raise DimensionMismatchError("NoisyOperator: vector length mismatch")
        z = self._plan.multiply(y) if self._plan is not None else denseMultiply(self._cloud, self._kernel, y,
                                                                                    self._diag)
        return z + self._noise * y


def cgSolve(op: NoisyOperator, rhs, tolerance: float, maxIterations: int,
            jacobiPreconditioner: bool = False, restartOnIncrease: bool = True) -> CgResult:
    """fkt::cgSolve (gp.cpp:58-124); the iterates live on the GPU (csrc/gp.cu).

    restartOnIncrease (additive, default = the reference): restart from the
    current iterate whenever the residual norm grows (gp.cpp:100-111). CG
    residuals are not monotone, so on smooth kernels the rule fires about every
    other iteration and the solve stalls -- exactly as in the reference;
    False runs textbook CG."""
    b = _f64(rhs).ravel()
    if b.size != op.size():
        raise DimensionMismatchError("cgSolve: rhs length mismatch")
    if not tolerance > 0.0:
        raise InvalidArgument("cgSolve requires a positive tolerance")
    x = np.empty(b.size)
    dg = _L.FktCgDiagnosticsC()
    if op._plan is not None:
        _check(lib.fkt_cg_solve(op._plan._h, _dptr(op._noise), _dptr(b), float(tolerance), int(maxIterations),
                                int(bool(jacobiPreconditioner)), int(bool(restartOnIncrease)), _dptr(x), C.byref(dg)))
    else:
        k, v, n = _params(op._kernel.parameters())
        cl = op._cloud
        _check(lib.fkt_cg_solve_dense(cl.n, cl.d, _dptr(cl.x), op._kernel.name().encode(), k, v, n,
                                      int(op._diag is not None), float(op._diag or 0.0), _dptr(op._noise), _dptr(b),
                                      float(tolerance), int(maxIterations), int(bool(jacobiPreconditioner)),
                                      int(bool(restartOnIncrease)), _dptr(x), C.byref(dg)))
    return CgResult(x, CgDiagnostics._from(dg))


@dataclass
class GpOptions:
    """fkt::GpOptions (gp.hpp:51-58)."""

    fkt: FktOptions = field(default_factory=FktOptions)
    cgTolerance: float = 1e-10
    cgMaxIterations: int = 1000
    jacobiPreconditioner: bool = False
    dense: bool = False
    priorMean: Optional[float] = None
    restartOnIncrease: bool = True  # additive; see cgSolve


@dataclass
class GpPrediction:
    """fkt::GpPrediction (gp.hpp:60-63)."""

    mean: np.ndarray
    diagnostics: CgDiagnostics


def gpPosteriorMean(train: PointCloud, y, noise, kernel: IsotropicKernel, test: PointCloud,
                    options: Optional[GpOptions] = None) -> GpPrediction:
    """fkt::gpPosteriorMean (gp.cpp:126-177) on the GPU."""
    o = options or GpOptions()
    y, noise = _f64(y).ravel(), _f64(noise).ravel()
    if y.size != train.n or noise.size != train.n:
        raise DimensionMismatchError("gpPosteriorMean: training vector lengths must match the cloud")
    if test.d != train.d:
        raise DimensionMismatchError("gpPosteriorMean: train/test dimension mismatch")
    oc = _L.FktGpOptionsC(o.fkt._c(), float(o.cgTolerance), int(o.cgMaxIterations), int(bool(o.jacobiPreconditioner)),
                          int(bool(o.dense)), int(o.priorMean is not None), float(o.priorMean or 0.0),
                          int(bool(o.restartOnIncrease)))
    mean = np.empty(test.n)
    dg = _L.FktCgDiagnosticsC()
    k, v, n = _params(kernel.parameters())
    tx = _f64(test.x) if test.n > 0 else np.zeros((1, train.d))
    _check(lib.fkt_gp_posterior_mean(train.n, train.d, _dptr(_f64(train.x)), _dptr(y), _dptr(noise),
                                     kernel.name().encode(), k, v, n, test.n, _dptr(tx), C.byref(oc),
                                     _dptr(mean) if test.n > 0 else None, C.byref(dg)))
    return GpPrediction(mean, CgDiagnostics._from(dg))


def expansionSize(d: int, p: int) -> int:
    r = lib.fkt_expansion_size(int(d), int(p))
    if r < 0:
        _check(lib.fkt_last_error_code())
    return int(r)


def tbar(d: int, p: int, k: int, j: int, m: int):
    """(double, 'num/den') of the exact coefficient T-bar_kjm (coefficients.hpp:47-52)."""
    v = C.c_double()
    buf = C.create_string_buffer(4096)
    _check(lib.fkt_tbar(d, p, k, j, m, C.byref(v), buf, 4096))
    return v.value, buf.value.decode()


class CoefficientTable:
    """fkt::CoefficientTable (coefficients.hpp:43-76): the exact T-bar table,
    its text serialization (coefficients.cpp:113-166) and equality."""

    def __init__(self, d: int, p: int):
        self._d, self._p = int(d), int(p)
        if self._p > 20:
            raise OrderTooLargeError(f"expansion order {p} exceeds the supported cap 20")

    def dimension(self) -> int:
        return self._d

    def maxOrder(self) -> int:
        return self._p

    def tbar(self, k: int, j: int, m: int) -> str:
        return tbar(self._d, self._p, k, j, m)[1]

    def tbarDouble(self, k: int, j: int, m: int) -> float:
        return tbar(self._d, self._p, k, j, m)[0]

    def serialize(self) -> str:
        need = lib.fkt_tbar_serialize(self._d, self._p, None, 0)
        if need < 0:
            _check(lib.fkt_last_error_code())
        buf = C.create_string_buffer(int(need))
        lib.fkt_tbar_serialize(self._d, self._p, buf, need)
        return buf.value.decode()

    @staticmethod
    def deserialize(text: str) -> Optional["CoefficientTable"]:
        """None when the text does not parse (as the reference's nullopt);
        the table's (d, p) otherwise. `equalsComputed` tells whether it equals
        the table computed here."""
        d, p, eq = C.c_int(), C.c_int(), C.c_int()
        if lib.fkt_tbar_deserialize(text.encode(), C.byref(d), C.byref(p), C.byref(eq)) != 0:
            return None
        t = CoefficientTable.__new__(CoefficientTable)
        t._d, t._p = d.value, p.value
        t.equalsComputed = bool(eq.value)
        return t

    def __eq__(self, other) -> bool:
        return isinstance(other, CoefficientTable) and self.serialize() == other.serialize()


def coefficientTable(d: int, p: int) -> CoefficientTable:
    """fkt::coefficientTable (coefficients.cpp:210-213); FKT_CACHE_DIR honoured."""
    return CoefficientTable(d, p)


def compressionRanks(kernel: IsotropicKernel, d: int, p: int):
    ranks = (C.c_int * (p + 1))()
    k, v, n = _params(kernel.parameters())
    _check(lib.fkt_compression_ranks(kernel.name().encode(), k, v, n, d, p, ranks))
    return list(ranks)


def additionNormalizer(d: int, k: int) -> float:
    return float(lib.fkt_addition_normalizer(d, k))


def configDims(cfg: int):
    d, r = C.c_int(), C.c_int()
    if lib.fkt_config_dims(cfg, C.byref(d), C.byref(r)) != 0:
        raise InvalidArgument("config must be 1..5")
    return d.value, r.value


def synthConfig(cfg: int, n: int, seed: int = 42):
    """SURVEY Appendix B inputs: (x [n x d], w [n] or [n x 16] column-major)."""
    d, nrhs = configDims(cfg)
    x = np.empty((n, d))
    w = np.empty((nrhs, n))
    _check(lib.fkt_synth_config(cfg, n, seed, _dptr(x), _dptr(w)))
    return x, (w[0] if nrhs == 1 else w.T)


def synthCloud(kind: str, n: int, d: int, seed: int, with_weights: bool = True):
    """fkt::Rng(seed) -> {cube,sphere,mixture}Cloud(n, d) then normalVector(n)."""
    x = np.empty((n, d))
    y = np.empty(n) if with_weights else None
    _check(lib.fkt_synth_cloud(kind.encode(), n, d, seed, _dptr(x), _dptr(y) if y is not None else None))
    return (x, y) if with_weights else x
