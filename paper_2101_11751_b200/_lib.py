"""ctypes binding of libgsgpc.so (the C ABI in include/gsgpc.h).

The product path has no fallback: if the in-tree CUDA library is missing or cannot be
loaded, importing the API raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libgsgpc.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "gsgpc.h")

OK, INVALID_ARGUMENT, OUT_OF_GRID, BREAKDOWN, NONCONVERGENCE, CUDA_ERROR, UNSUPPORTED, RUNTIME_ERROR = range(8)
LINEAR, CUBIC = 0, 1
F32, F64 = 0, 1
MAX_DIM = 3


class Grid_t(C.Structure):
    _fields_ = [("dim", C.c_int32), ("min", C.c_double * MAX_DIM), ("max", C.c_double * MAX_DIM),
                ("size", C.c_int64 * MAX_DIM)]


class Points_t(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("x", C.c_void_p), ("x_row_stride", C.c_int64),
                ("x_col_offset", C.c_int64 * MAX_DIM), ("y", C.c_void_p), ("y_stride", C.c_int64)]


class SolveInfo_t(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("residual_sq", C.c_double),
                ("loop_seconds", C.c_double)]


class LoglikOptions_t(C.Structure):
    _fields_ = [("solve_tol", C.c_double), ("probes", C.c_int32), ("max_depth", C.c_int32),
                ("quad_tol", C.c_double), ("seed", C.c_uint64), ("maxiter", C.c_int32), ("route", C.c_int32),
                ("dense_cap", C.c_int64), ("probe_begin", C.c_int32), ("probe_end", C.c_int32)]


class LoglikResult_t(C.Structure):
    _fields_ = [("loglik", C.c_double), ("logdet_term", C.c_double), ("quad_term", C.c_double),
                ("const_term", C.c_double), ("probes_used", C.c_int32), ("solver_iterations", C.c_int32),
                ("max_depth_used", C.c_int32), ("logdet_route", C.c_int32), ("slq_sum", C.c_double),
                ("slq_count", C.c_int32), ("logdet_shift", C.c_double)]


_vp, _i, _i64, _d = C.c_void_p, C.c_int, C.c_int64, C.c_double
_P = C.POINTER

SIGNATURES = {
    "gsgpc_version": (C.c_char_p, []),
    "gsgpc_ctx_create": (_i, [_i, _P(_vp)]),
    "gsgpc_group_create": (_i, [_P(_i), _i, _P(_vp)]),
    "gsgpc_group_destroy": (_i, [_vp]),
    "gsgpc_group_info": (_i, [_vp, _P(_i), _P(_i)]),
    "gsgpc_group_ctx": (_vp, [_vp, _i]),
    "gsgpc_group_last_error": (C.c_char_p, [_vp]),
    "gsgpc_group_last_error_row": (_i64, [_vp]),
    "gsgpc_group_sufficient_stats": (_i, [_vp, _P(Grid_t), _i, _P(Points_t), _i64, _i, C.c_uint64, _P(_vp)]),
    "gsgpc_group_allreduce_stats": (_i, [_vp, _P(_vp)]),
    "gsgpc_ctx_destroy": (None, [_vp]),
    "gsgpc_ctx_set_stream": (_i, [_vp, _vp]),
    "gsgpc_ctx_stream": (_vp, [_vp]),
    "gsgpc_ctx_synchronize": (_i, [_vp]),
    "gsgpc_last_error": (C.c_char_p, [_vp]),
    "gsgpc_last_error_row": (_i64, [_vp]),
    "gsgpc_ctx_launch_count": (C.c_uint64, [_vp]),
    "gsgpc_ctx_enable_phase_timing": (_i, [_vp, _i]),
    "gsgpc_ctx_phase_times": (_i, [_vp, _vp, _vp]),
    "gsgpc_ctx_reset_phase_times": (_i, [_vp]),
    "gsgpc_fit_grid_to_data": (_i, [_i, _vp, _vp, _vp, _i, _P(Grid_t)]),
    "gsgpc_interp_weights": (_i, [_vp, _P(Grid_t), _i, _P(Points_t), _i64, _vp, _vp, _vp, _vp]),
    "gsgpc_stats_create": (_i, [_vp, _P(Grid_t), _i, _P(_vp)]),
    "gsgpc_stats_destroy": (None, [_vp]),
    "gsgpc_stats_add": (_i, [_vp, _vp, _P(Points_t), _i64, _vp, _i]),
    "gsgpc_stats_add_file": (_i, [_vp, _vp, C.c_char_p, _P(_i64)]),
    "gsgpc_stats_merge": (_i, [_vp, _vp, _vp]),
    "gsgpc_stats_reset": (_i, [_vp, _vp]),
    "gsgpc_stats_enable_probes": (_i, [_vp, _vp, _i, C.c_uint64]),
    "gsgpc_stats_enable_probes_at": (_i, [_vp, _vp, _i, C.c_uint64, _i64]),
    "gsgpc_probe_stream_bits": (_i, [C.c_uint64, C.c_uint64, C.c_uint64, _i64, _vp]),
    "gsgpc_diag_fp64_peak": (_i, [_vp, _P(_d)]),
    "gsgpc_diag_fp64_tensor": (_i, [_vp, _P(_d), _P(_d)]),
    "gsgpc_stats_finalize": (_i, [_vp, _vp]),
    "gsgpc_sufficient_stats": (_i, [_vp, _P(Grid_t), _i, _P(Points_t), _i64, _P(_vp)]),
    "gsgpc_stats_info": (_i, [_vp, _vp, _P(_i64), _P(_i64), _P(_d), _P(_i64), _P(C.c_int32)]),
    "gsgpc_stats_grid": (_i, [_vp, _P(Grid_t), _P(_i)]),
    "gsgpc_stats_copy_wty": (_i, [_vp, _vp, _vp]),
    "gsgpc_stats_copy_stencil": (_i, [_vp, _vp, _vp, _vp]),
    "gsgpc_stats_copy_probe_images": (_i, [_vp, _vp, _vp]),
    "gsgpc_stats_csr_nnz": (_i, [_vp, _vp, _P(_i64), _P(_i64)]),
    "gsgpc_stats_export_csr": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "gsgpc_stats_apply_wtw": (_i, [_vp, _vp, _vp, _vp]),
    "gsgpc_stats_reduce_buffer": (_i, [_vp, _vp, _P(_vp), _P(_i64)]),
    "gsgpc_stats_pattern_buffer": (_i, [_vp, _vp, _P(_vp), _P(_i64)]),
    "gsgpc_stats_mark_reduced": (_i, [_vp, _vp]),
    "gsgpc_stats_save": (_i, [_vp, _vp, C.c_char_p]),
    "gsgpc_stats_load": (_i, [_vp, C.c_char_p, _P(_vp)]),
    "gsgpc_kg_create": (_i, [_vp, _P(Grid_t), _vp, _d, _d, _P(_vp)]),
    "gsgpc_kg_create_ex": (_i, [_vp, _P(Grid_t), _vp, _d, _d, _i64, _P(_vp)]),
    "gsgpc_next_fast_fft_size": (_i64, [_i64]),
    "gsgpc_kg_destroy": (None, [_vp]),
    "gsgpc_kg_apply": (_i, [_vp, _vp, _vp, _vp]),
    "gsgpc_kg_info": (_i, [_vp, _P(_i64), _P(_d)]),
    "gsgpc_factorized_cg_grid_rhs": (_i, [_vp, _vp, _vp, _vp, _d, _d, _d, _i, _vp, _P(SolveInfo_t), _vp, _vp, _vp]),
    "gsgpc_posterior_mean_gsgp": (_i, [_vp, _vp, _vp, _d, _d, _i, _vp, _P(SolveInfo_t)]),
    "gsgpc_predict_mean": (_i, [_vp, _P(Grid_t), _i, _vp, _P(Points_t), _i64, _vp]),
    "gsgpc_factorized_lanczos_fused": (_i, [_vp, _vp, _vp, _i, _vp, _vp, _vp, _d, _i, _vp, _vp, _vp]),
    "gsgpc_posterior_cov_exact": (_i, [_vp, _vp, _vp, _d, _P(Points_t), _i64, _d, _i, _vp, _P(_d), _P(C.c_int32)]),
    "gsgpc_posterior_cov_lowrank": (_i, [_vp, _vp, _vp, _d, _i64, _P(_vp)]),
    "gsgpc_lowrank_destroy": (None, [_vp]),
    "gsgpc_lowrank_rank": (_i, [_vp, _P(_i64)]),
    "gsgpc_lowrank_cov_matrix": (_i, [_vp, _vp, _P(Points_t), _i64, _vp]),
    "gsgpc_lowrank_query": (_i, [_vp, _vp, _vp, _vp, _P(_d)]),
    "gsgpc_log_likelihood_gsgp": (_i, [_vp, _vp, _vp, _d, _P(LoglikOptions_t), _P(LoglikResult_t)]),
}


def header_symbols(path: str = HEADER):
    """Function names declared in include/gsgpc.h."""
    txt = open(path).read()
    return sorted(set(re.findall(r"\b(gsgpc_[a-z0-9_]+)\s*\(", txt)))


_lib = None


def load(path: str = LIB_PATH):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libgsgpc.so not built at {path}: run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    L = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
