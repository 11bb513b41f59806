"""ctypes binding of the C-ABI in include/nlgpu.h (libnlgpu.so).

The native library is REQUIRED: importing this module on a machine where the
library is missing raises immediately — there is no Python or CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libnlgpu.so")

NLG_OK, NLG_EINVAL, NLG_EDOMAIN, NLG_ERANGE, NLG_ERUNTIME, NLG_ECUDA, NLG_ENCCL, NLG_EUNSUPPORTED = range(8)
LEAF, POINT = 0, 1
MASS, DIFFERENCE = 0, 1
CLIP, COLLAR = 0, 1
TRUNCATED, INVERSE_S, CONICAL, KAPPA, FRACTIONAL, PERIDYNAMIC = range(6)
ROUTE_TRUNCATED, ROUTE_SMOOTH, ROUTE_FULL = range(3)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)


class Desc(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("n", C.c_int64), ("family", C.c_int), ("route", C.c_int),
        ("poly", _dp), ("npoly", C.c_int), ("tail", _dp), ("ntail", C.c_int), ("order", C.c_int),
        ("c", C.c_double), ("alpha", C.c_double), ("rule", C.c_int), ("form", C.c_int),
        ("exterior", C.c_int), ("divergence", C.c_int), ("delta", _dp), ("delta0", C.c_double),
        ("reach", C.c_double), ("coeff", _dp), ("coeff0", C.c_double), ("kappa", _dp),
        ("row_begin", C.c_int64), ("row_end", C.c_int64), ("device", C.c_int),
    ]


class SolveReport(C.Structure):
    _fields_ = [("method", C.c_int), ("converged", C.c_int), ("iterations", C.c_int64),
                ("final_residual", C.c_double)]


SOLVE_CG, SOLVE_CGNR, SOLVE_DIRECT = 0, 1, 0x10


class Info(C.Structure):
    _fields_ = [("halo_lo", C.c_int64), ("halo_hi", C.c_int64), ("n_in", C.c_int64),
                ("n_out", C.c_int64), ("fast_method", C.c_int), ("exp_terms", C.c_int),
                ("near_cells", C.c_int), ("far_rel_err", C.c_double), ("fft_len", C.c_int64),
                ("fft_rows", C.c_int)]


EXPORTS = {
    "nlg_halo_rows": ([C.POINTER(Desc), C.c_double, _ip], C.c_int),
    "nlg_plan_create": ([C.POINTER(Desc), C.POINTER(C.c_void_p)], C.c_int),
    "nlg_plan_destroy": ([C.c_void_p], None),
    "nlg_plan_info": ([C.c_void_p, C.POINTER(Info)], C.c_int),
    "nlg_apply_fast": ([C.c_void_p, _dp, _dp], C.c_int),
    "nlg_apply_direct": ([C.c_void_p, _dp, _dp, _ip], C.c_int),
    "nlg_apply_fast_dev": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "nlg_apply_direct_dev": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "nlg_apply_direct_at": ([C.c_void_p, _dp, _ip, C.c_int64, _dp, _ip], C.c_int),
    "nlg_counters": ([C.c_void_p, _ip, _ip], C.c_int),
    "nlg_set_profiling": ([C.c_void_p, C.c_int], C.c_int),
    "nlg_apply_fast_dev_begin": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "nlg_apply_fast_dev_end": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "nlg_stage_times": ([C.c_void_p, _dp, _ip, C.POINTER(C.c_int)], C.c_int),
    "nlg_group_create": ([C.POINTER(Desc), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)], C.c_int),
    "nlg_group_destroy": ([C.c_void_p], None),
    "nlg_group_info": ([C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), _ip, _ip, _ip], C.c_int),
    "nlg_group_apply_fast": ([C.c_void_p, _dp, _dp], C.c_int),
    "nlg_group_apply_fast_dev": ([C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)], C.c_int),
    "nlg_group_last_error": ([], C.c_char_p),
    "nlg_launch_count": ([C.c_void_p, _ip], C.c_int),
    "nlg_match_polynomial": ([C.c_int, C.c_double, _dp], C.c_int),
    "nlg_match_polynomial_exact": ([C.c_int, _ip, _ip], C.c_int),
    "nlg_split": ([C.c_int, C.c_double, _dp, _dp, C.POINTER(C.c_int)], C.c_int),
    "nlg_expsum_fit": ([C.c_double, C.c_int, C.c_int64, _dp, _dp, C.POINTER(C.c_int), _dp], C.c_int),
    "nlg_apply_transpose": ([C.c_void_p, _dp, _dp], C.c_int),
    "nlg_apply_transpose_dev": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "nlg_assemble_dense": ([C.c_void_p, _dp], C.c_int),
    "nlg_solve_dirichlet": ([C.c_void_p, _dp, C.c_double, C.c_int64, C.c_int, _dp, C.POINTER(SolveReport)],
                            C.c_int),
    "nlg_expsum_fit_narrow": ([C.c_double, C.c_int64, C.c_int64, C.c_double, C.c_int, _dp, _dp,
                               C.POINTER(C.c_int), _dp], C.c_int),
    "nlg_tree_decompose": ([C.c_int, C.c_int64, _dp, C.c_double, C.c_int64, C.POINTER(C.c_int), _ip, _ip, _ip],
                           C.c_int),
    "nlg_tree_count": ([C.c_int, C.c_int64, _dp, _ip, _ip], C.c_int),
    "nlg_tree_moments": ([C.c_int, C.c_int64, C.c_int, _dp, _dp, _ip], C.c_int),
    "nlg_last_error": ([], C.c_char_p),
    "nlg_abi_version": ([], C.c_int),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"native library missing: {LIB_PATH} — run `python -m paper_1905_08375_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in EXPORTS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


class NonlocError(RuntimeError):
    pass


def check(status: int, group: bool = False) -> None:
    if status == NLG_OK:
        return
    msg = (lib().nlg_group_last_error() if group else lib().nlg_last_error()).decode()
    if status in (NLG_EINVAL, NLG_EUNSUPPORTED):
        raise ValueError(msg)            # std::invalid_argument
    if status == NLG_EDOMAIN:
        raise ArithmeticError(msg)       # std::domain_error
    if status == NLG_ERANGE:
        raise IndexError(msg)            # std::out_of_range
    raise NonlocError(f"[status {status}] {msg}")   # std::runtime_error


def dptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


STAGES = ["direct", "span_scan", "span_eval", "es_aggregate", "es_carry", "es_main", "es_combine", "stencil",
          "es_fft", "box_fft", "box_ties", "box_pa_rows_fwd", "box_pb_cols_fwd", "box_pc_zstencil",
          "box_pd_cols_inv", "box_pe_rows_inv", "es_fft_p1_cols_fwd", "es_fft_p2_rows",
          "es_fft_p3_cols_inv"]   # plan.hpp enum Stage (kNumStages slots)
