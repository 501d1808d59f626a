"""ctypes binding of the C-ABI in include/fkt_cuda.h (lib/libfkt_cuda.so).

The shared library is built in-tree (``make -C paper_2106_04487_b200`` or
``__graft_entry__.build()``). There is no CPU fallback: if the library is
missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# FKTB_LIB_PATH: developer A/B knob (a variant build of the same library)
LIB_PATH = os.environ.get("FKTB_LIB_PATH") or os.path.join(_HERE, "lib", "libfkt_cuda.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C {_HERE}` (the FKT MVM has no CPU fallback)"
    )

lib = C.CDLL(LIB_PATH)

_d = C.POINTER(C.c_double)
_u32 = C.POINTER(C.c_uint32)
_i32 = C.POINTER(C.c_int)
_i64 = C.POINTER(C.c_int64)
_ll = C.POINTER(C.c_longlong)
_cstrs = C.POINTER(C.c_char_p)


class FktOptionsC(C.Structure):
    _fields_ = [
        ("p", C.c_int),
        ("theta", C.c_double),
        ("leaf_capacity", C.c_int),
        ("compression", C.c_int),
        ("eager_operators", C.c_int),
        ("barnes_hut", C.c_int),
        ("threads", C.c_int),
        ("has_diagonal", C.c_int),
        ("diagonal", C.c_double),
        ("near_precision", C.c_int),
        ("deterministic", C.c_int),
    ]


class FktCgDiagnosticsC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("final_residual", C.c_double), ("converged", C.c_int),
                ("restarts", C.c_int)]


class FktGpOptionsC(C.Structure):
    _fields_ = [("fkt", FktOptionsC), ("cg_tolerance", C.c_double), ("cg_max_iterations", C.c_int),
                ("jacobi", C.c_int), ("dense", C.c_int), ("has_prior_mean", C.c_int), ("prior_mean", C.c_double),
                ("restart_on_increase", C.c_int)]


class FktPlanInfoC(C.Structure):
    _fields_ = [
        ("n", C.c_int),
        ("d", C.c_int),
        ("p", C.c_int),
        ("nodes", C.c_longlong),
        ("leaves", C.c_longlong),
        ("depth", C.c_longlong),
        ("far_total", C.c_longlong),
        ("near_total", C.c_longlong),
        ("coefficient_count", C.c_longlong),
        ("stored_coefficients", C.c_longlong),
        ("compressed", C.c_int),
        ("plan_seconds", C.c_double),
        ("far_tiles", C.c_longlong),
        ("near_tiles", C.c_longlong),
        ("s2m_tiles", C.c_longlong),
        ("m2t_cartesian", C.c_int),
    ]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


# Every symbol declared in include/fkt_cuda.h, with its signature.
SIGNATURES = {
    "fkt_last_error": (C.c_char_p,),
    "fkt_last_error_code": (C.c_int,),
    "fkt_version": (C.c_char_p,),
    "fkt_kernel_count": (C.c_int,),
    "fkt_kernel_name": (C.c_char_p, C.c_int),
    "fkt_kernel_check": (C.c_int, C.c_char_p, _cstrs, _d, C.c_int, _i32, _i32, _d),
    "fkt_kernel_eval": (C.c_int, C.c_char_p, _cstrs, _d, C.c_int, _d, _d, C.c_longlong, C.c_int, C.c_double),
    "fkt_default_options": (None, C.POINTER(FktOptionsC)),
    "fkt_kernel_eval_jet": (C.c_int, C.c_char_p, _cstrs, _d, C.c_int, C.c_double, C.c_int, _d, _d),
    "fkt_kernel_recurrence": (C.c_int, C.c_char_p, _cstrs, _d, C.c_int, _i32, _i32, C.c_int, C.c_char_p, C.c_longlong),
    "fkt_plan_create": (C.c_int, C.c_int, C.c_int, _d, C.c_char_p, _cstrs, _d, C.c_int,
                        C.POINTER(FktOptionsC), C.POINTER(C.c_void_p)),
    "fkt_plan_destroy": (C.c_int, C.c_void_p),
    "fkt_plan_rebuild": (C.c_int, C.c_void_p, _d),
    "fkt_plan_rebuild_device": (C.c_int, C.c_void_p, C.c_void_p),
    "fkt_plan_multiply_sharded": (C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p),
    "fkt_nccl_unique_id": (C.c_int, C.c_char_p),
    "fkt_nccl_comm_create": (C.c_int, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)),
    "fkt_nccl_comm_destroy": (C.c_int, C.c_void_p),
    "fkt_plan_cache_get": (C.c_int, C.c_int, C.c_int, _d, C.c_char_p, _cstrs, _d, C.c_int, C.POINTER(FktOptionsC),
                           C.POINTER(C.c_void_p), _i32),
    "fkt_plan_cache_release": (C.c_int, C.c_void_p),
    "fkt_plan_cache_set_capacity": (C.c_int, C.c_int),
    "fkt_plan_cache_size": (C.c_int,),
    "fkt_plan_info_get": (C.c_int, C.c_void_p, C.POINTER(FktPlanInfoC)),
    "fkt_plan_multiply": (C.c_int, C.c_void_p, _d, _d, C.c_int),
    "fkt_plan_multiply_device": (C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p),
    "fkt_plan_stage_device": (C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p),
    "fkt_plan_set_shard": (C.c_int, C.c_void_p, C.c_int, C.c_int),
    "fkt_plan_shard_range": (C.c_int, C.c_void_p, _ll, _ll),
    "fkt_plan_moments_device": (C.c_int, C.c_void_p, C.POINTER(C.POINTER(C.c_double)), _ll),
    "fkt_default_gp_options": (None, C.POINTER(FktGpOptionsC)),
    "fkt_cg_solve": (C.c_int, C.c_void_p, _d, _d, C.c_double, C.c_int, C.c_int, C.c_int, _d,
                     C.POINTER(FktCgDiagnosticsC)),
    "fkt_cg_solve_dense": (C.c_int, C.c_int, C.c_int, _d, C.c_char_p, _cstrs, _d, C.c_int, C.c_int, C.c_double, _d, _d,
                           C.c_double, C.c_int, C.c_int, C.c_int, _d, C.POINTER(FktCgDiagnosticsC)),
    "fkt_gp_posterior_mean": (C.c_int, C.c_int, C.c_int, _d, _d, _d, C.c_char_p, _cstrs, _d, C.c_int, C.c_int, _d,
                              C.POINTER(FktGpOptionsC), _d, C.POINTER(FktCgDiagnosticsC)),
    "fkt_plan_kernel_launches": (C.c_longlong, C.c_void_p, C.c_int),
    "fkt_plan_near_forms": (C.c_int, C.c_void_p, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)),
    "fkt_shard_cuts": (C.c_int, _u32, C.POINTER(C.c_ulonglong), C.c_int, C.c_int, C.c_uint32, _u32),
    "fkt_plan_tree": (C.c_void_p, C.c_void_p),
    "fkt_tree_create": (C.c_int, C.c_int, C.c_int, _d, C.c_int, C.POINTER(C.c_void_p)),
    "fkt_tree_compute_sets": (C.c_int, C.c_void_p, C.c_double),
    "fkt_tree_destroy": (C.c_int, C.c_void_p),
    "fkt_tree_sizes": (C.c_int, C.c_void_p, _ll, _ll, _ll, _ll, _d),
    "fkt_tree_nodes": (C.c_int, C.c_void_p, _u32, _u32, _i32, _i32, _d, _d, _d, _d),
    "fkt_tree_order": (C.c_int, C.c_void_p, _u32),
    "fkt_tree_points": (C.c_int, C.c_void_p, _d),
    "fkt_tree_far_sets": (C.c_int, C.c_void_p, _ll, _u32),
    "fkt_tree_near_sets": (C.c_int, C.c_void_p, _ll, _u32),
    "fkt_dense_multiply": (C.c_int, C.c_int, C.c_int, _d, C.c_char_p, _cstrs, _d, C.c_int, _d, _d, C.c_int,
                           C.c_double),
    "fkt_dense_rows": (C.c_int, C.c_int, C.c_int, _d, C.c_char_p, _cstrs, _d, C.c_int, _d, C.c_int, _i64, _d,
                       C.c_int, C.c_double),
    "fkt_relative_error": (C.c_int, _d, _d, C.c_longlong, _d),
    "fkt_expansion_size": (C.c_longlong, C.c_int, C.c_int),
    "fkt_tbar": (C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _d, C.c_char_p, C.c_int),
    "fkt_tbar_serialize": (C.c_longlong, C.c_int, C.c_int, C.c_char_p, C.c_longlong),
    "fkt_tbar_deserialize": (C.c_int, C.c_char_p, _i32, _i32, _i32),
    "fkt_compression_ranks": (C.c_int, C.c_char_p, _cstrs, _d, C.c_int, C.c_int, C.c_int, _i32),
    "fkt_addition_normalizer": (C.c_double, C.c_int, C.c_int),
    "fkt_harmonic_count": (C.c_longlong, C.c_int, C.c_int),
    "fkt_fma_peak": (C.c_int, C.c_int, _d),
    "fkt_fp64_peaks": (C.c_int, _d, _d),
    "fkt_plan_phases": (C.c_int, C.c_void_p, _d, C.c_int),
    "fkt_synth_cloud": (C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_uint64, _d, _d),
    "fkt_synth_config": (C.c_int, C.c_int, C.c_int, C.c_uint64, _d, _d),
    "fkt_config_dims": (C.c_int, C.c_int, _i32, _i32),
}

for _name, (_res, *_args) in SIGNATURES.items():
    _sig(_name, _res, *_args)
