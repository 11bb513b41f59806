"""oracle/oracle.py — ctypes loaders for the CPU checkers.

TEST INFRASTRUCTURE ONLY. Importable from tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline leg, --impl reference) — never from the product package.

Two libraries:
  * ``_build/liborc.so`` — the restated C oracle (nonloc_oracle.c), always
    buildable (gcc) and present on the GPU box (built in-tree, shipped by gpurun);
  * ``_ref/libnonloc_ref.so`` — the reference itself, compiled from the
    unmodified sources under /root/reference/proj by ``make ref``; present only
    where it was built (it travels to the GPU box as a prebuilt file).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "_build", "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libnonloc_ref.so")
REF_SRC = "/root/reference/proj"

LEAF, POINT = 0, 1
MASS, DIFFERENCE = 0, 1
CLIP, COLLAR = 0, 1
TRUNCATED, INVERSE_S, CONICAL, KAPPA, FRACTIONAL, PERIDYNAMIC = range(6)
ROUTE_TRUNCATED, ROUTE_SMOOTH, ROUTE_FULL = range(3)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)


class OrcDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("n", C.c_int64), ("family", C.c_int), ("route", C.c_int),
        ("poly", _dp), ("npoly", C.c_int), ("tail", _dp), ("ntail", C.c_int),
        ("order", C.c_int), ("c", C.c_double), ("alpha", C.c_double),
        ("rule", C.c_int), ("form", C.c_int), ("exterior", C.c_int),
        ("divergence", C.c_int), ("delta", _dp), ("delta0", C.c_double),
        ("reach", C.c_double), ("coeff", _dp), ("coeff0", C.c_double), ("kappa", _dp),
    ]


def build(ref: bool | None = None) -> None:
    """Compile liborc.so (and oracle/_ref when the reference sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_SO):
            build(ref=False)
        lib = C.CDLL(ORC_SO)
        lib.orc_apply.argtypes = [C.POINTER(OrcDesc), _dp, _dp, _ip, C.c_int64, _ip]
        lib.orc_apply_peri.argtypes = [C.POINTER(OrcDesc), _dp, _dp, _ip, C.c_int64, _ip]
        lib.orc_random_vector.argtypes = [C.c_int64, C.c_uint64, _dp]
        lib.orc_match_polynomial.argtypes = [C.c_int, C.c_double, _dp]
        lib.orc_bump_horizon.argtypes = [C.c_int, C.c_int64, C.c_double, _dp]
        lib.orc_leaf_in.argtypes = [C.c_int, C.c_int64, _ip, _ip, C.c_double]
        lib.orc_point_in.argtypes = [C.c_int, C.c_int64, _ip, _ip, C.c_double]
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError("oracle/_ref/libnonloc_ref.so not built (needs /root/reference)")
        lib = C.CDLL(REF_SO)
        i, d = C.c_int, C.c_double
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_random_vector.argtypes = [C.c_int64, C.c_uint64, _dp]
        lib.ref_match_polynomial.argtypes = [i, d, _dp]
        lib.ref_split.argtypes = [i, d, _dp, _dp, C.POINTER(C.c_int)]
        lib.ref_kappa.argtypes = [i, d, C.c_int64, _dp, _dp]
        lib.ref_truncated_fast.argtypes = [i, i, i, i, d, d, _dp, _dp, _ip, _dp, i]
        lib.ref_truncated_dense.argtypes = [i, i, i, i, d, d, i, i, _dp, _dp, _ip]
        lib.ref_smooth_dense.argtypes = [i, i, i, i, d, d, _dp, _dp, _ip]
        lib.ref_full_dense.argtypes = [i, i, i, i, i, d, d, i, _dp, _dp, _ip]
        lib.ref_apply_split.argtypes = [i, i, i, i, d, d, i, _dp, _dp]
        lib.ref_full_dense_general.argtypes = [i, i, _dp, d, _dp, _dp, d, _dp, _dp, _ip]
        lib.ref_full_dense_general_at.argtypes = [i, i, _dp, d, _dp, _dp, d, _dp, _ip, C.c_int64,
                                                  _dp, i, _ip]
        lib.ref_assemble_dense.argtypes = [i, i, i, i, i, d, d, i, i, i, _dp]
        lib.ref_solve_truncated.argtypes = [i, i, i, i, d, d, _dp, d, C.c_int64, i, _dp, _ip, _dp,
                                            C.POINTER(C.c_int), C.POINTER(C.c_int)]
        lib.ref_dense_direct_solve.argtypes = [C.c_int64, _dp, _dp, _dp]
        lib.ref_decompose.argtypes = [i, i, _dp, d, C.c_int64, C.POINTER(C.c_int), _ip, _ip, _ip]
        lib.ref_count_recur_calls.argtypes = [i, i, _dp, _ip]
        lib.ref_moments.argtypes = [i, i, i, _dp, _dp, _ip]
        _ref = lib
    return _ref


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _check_ref(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {ref().ref_last_error().decode()}")


# ----------------------------------------------------------------------------
# restated oracle wrappers
# ----------------------------------------------------------------------------

def random_vector(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    orc().orc_random_vector(n, seed, _p(out))
    return out


def match_polynomial(K: int, c: float = 1.0) -> np.ndarray:
    out = np.empty(K + 1, dtype=np.float64)
    if orc().orc_match_polynomial(K, c, _p(out)) != 0:
        raise ValueError("matching order out of range")
    return out


def bump_horizon(dim: int, n: int, delta0: float) -> np.ndarray:
    out = np.empty(n ** dim, dtype=np.float64)
    orc().orc_bump_horizon(dim, n, delta0, _p(out))
    return out


def apply(dim, n, u, *, family=FRACTIONAL, route=ROUTE_FULL, poly=None, tail=None,
          order=0, c=1.0, alpha=1.0, rule=POINT, form=DIFFERENCE, exterior=CLIP,
          divergence=False, delta=None, delta0=0.0, reach=0.0, coeff=None, coeff0=1.0,
          kappa=None, targets=None, peri=False):
    """Direct-sum oracle; returns (out, pairs)."""
    keep = []

    def arr(a):
        if a is None:
            return None
        a = np.ascontiguousarray(a, dtype=np.float64)
        keep.append(a)
        return a

    poly, tail, delta, coeff, kappa = map(arr, (poly, tail, delta, coeff, kappa))
    u = np.ascontiguousarray(u, dtype=np.float64)
    desc = OrcDesc(dim, n, family, route, _p(poly), 0 if poly is None else len(poly),
                   _p(tail), 0 if tail is None else len(tail), order, c, alpha, rule, form,
                   exterior, int(divergence), _p(delta), delta0, reach, _p(coeff), coeff0,
                   _p(kappa))
    N = n ** dim
    tg = None
    cnt = N
    if targets is not None:
        tg = np.ascontiguousarray(targets, dtype=np.int64)
        cnt = len(tg)
    pairs = C.c_int64(0)
    if peri:
        out = np.empty(dim * cnt, dtype=np.float64)
        rc = orc().orc_apply_peri(C.byref(desc), _p(u), _p(out),
                                  None if tg is None else tg.ctypes.data_as(_ip),
                                  cnt if tg is not None else 0, C.byref(pairs))
    else:
        out = np.empty(cnt, dtype=np.float64)
        rc = orc().orc_apply(C.byref(desc), _p(u), _p(out),
                             None if tg is None else tg.ctypes.data_as(_ip),
                             cnt if tg is not None else 0, C.byref(pairs))
    if rc != 0:
        raise ValueError(f"oracle error {rc}")
    return out, pairs.value


# ----------------------------------------------------------------------------
# compiled-reference wrappers (names follow the reference API)
# ----------------------------------------------------------------------------

def ref_random_vector(n, seed):
    out = np.empty(n, dtype=np.float64)
    _check_ref(ref().ref_random_vector(n, seed, _p(out)))
    return out


def ref_match_polynomial(K, c=1.0):
    out = np.empty(K + 1, dtype=np.float64)
    _check_ref(ref().ref_match_polynomial(K, c, _p(out)))
    return out


def ref_split(K, c=1.0):
    poly = np.empty(K + 1)
    tail = np.empty(2 * K + 4)
    nt = C.c_int(0)
    _check_ref(ref().ref_split(K, c, _p(poly), _p(tail), C.byref(nt)))
    return poly, tail[: nt.value].copy()


def ref_kappa(K, s, c=1.0):
    s = np.ascontiguousarray(s, dtype=np.float64)
    out = np.empty_like(s)
    _check_ref(ref().ref_kappa(K, c, len(s), _p(s), _p(out)))
    return out


def ref_truncated_fast(dim, n, K, horizon_kind, delta0, u, coeff=1.0, reps=1):
    """TruncatedOperator(spec, grid).apply(u); returns (out, counters, times)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    cnt = np.zeros(3, dtype=np.int64)
    tm = np.zeros(2)
    _check_ref(ref().ref_truncated_fast(dim, n, K, horizon_kind, delta0, coeff, _p(u), _p(out),
                                        cnt.ctypes.data_as(_ip), _p(tm), reps))
    return out, cnt, tm


def ref_truncated_dense(dim, n, K, horizon_kind, delta0, u, rule=LEAF, form=MASS, coeff=1.0):
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    pairs = C.c_int64(0)
    _check_ref(ref().ref_truncated_dense(dim, n, K, horizon_kind, delta0, coeff, rule, form,
                                         _p(u), _p(out), C.byref(pairs)))
    return out, pairs.value


def ref_smooth_dense(dim, n, K, horizon_kind, delta0, u, coeff=1.0):
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    pairs = C.c_int64(0)
    _check_ref(ref().ref_smooth_dense(dim, n, K, horizon_kind, delta0, coeff, _p(u), _p(out),
                                      C.byref(pairs)))
    return out, pairs.value


def ref_full_dense(dim, n, family, order, horizon_kind, delta0, u, coeff=1.0, divergence=False):
    """family: 0 InverseS, 1 Conical, 2 Regularized(order), 3 Truncated(order)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    pairs = C.c_int64(0)
    _check_ref(ref().ref_full_dense(dim, n, family, order, horizon_kind, delta0, coeff,
                                    int(divergence), _p(u), _p(out), C.byref(pairs)))
    return out, pairs.value


def ref_apply_split(dim, n, K, horizon_kind, delta0, u, truncated=0, coeff=1.0):
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    _check_ref(ref().ref_apply_split(dim, n, K, horizon_kind, delta0, coeff, truncated,
                                     _p(u), _p(out)))
    return out


def ref_full_dense_general(dim, n, delta, cx, kappa, alpha, u):
    u = np.ascontiguousarray(u, dtype=np.float64)
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    cx = None if cx is None else np.ascontiguousarray(cx, dtype=np.float64)
    kappa = None if kappa is None else np.ascontiguousarray(kappa, dtype=np.float64)
    out = np.empty_like(u)
    pairs = C.c_int64(0)
    _check_ref(ref().ref_full_dense_general(dim, n, _p(delta), float(delta.max()), _p(cx),
                                            _p(kappa), alpha, _p(u), _p(out), C.byref(pairs)))
    return out, pairs.value


def ref_full_dense_general_at(dim, n, delta, cx, kappa, alpha, u, targets, nthreads=1,
                              delta_max=None):
    """The reference's apply_full_dense inner loop + eval_omega at selected
    targets (threaded); returns (out, pairs)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    cx = None if cx is None else np.ascontiguousarray(cx, dtype=np.float64)
    kappa = None if kappa is None else np.ascontiguousarray(kappa, dtype=np.float64)
    tg = np.ascontiguousarray(targets, dtype=np.int64)
    out = np.empty(len(tg))
    pairs = C.c_int64(0)
    dm = float(delta.max()) if delta_max is None else float(delta_max)
    _check_ref(ref().ref_full_dense_general_at(dim, n, _p(delta), dm, _p(cx), _p(kappa), alpha,
                                               _p(u), tg.ctypes.data_as(_ip), len(tg), _p(out),
                                               nthreads, C.byref(pairs)))
    return out, pairs.value


def rel_inf(a, b) -> float:
    """The reference's parity metric max|a-b| / max|b| (bench.cpp:61-67)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.max(np.abs(b)) if b.size else 0.0
    num = np.max(np.abs(a - b)) if b.size else 0.0
    return float(num / den) if den > 0 else float(num)


def ref_assemble_dense(dim, n, family, order, horizon_kind, delta0, rule=LEAF, form=MASS, coeff=1.0,
                       divergence=False):
    """assemble_dense_matrix (operators.cpp:262-303); family 3 = truncated K=order."""
    N = n ** dim
    a = np.empty(N * N)
    _check_ref(ref().ref_assemble_dense(dim, n, family, order, horizon_kind, delta0, coeff, int(divergence),
                                        rule, form, _p(a)))
    return a


def ref_solve_truncated(dim, n, K, horizon_kind, delta0, f, tol, max_iter, use_dense=False, coeff=1.0):
    """The reference's cmd_solve path (tools/nonloc_main.cpp:189-222):
    returns (u, iterations, final_residual, converged, method)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    u = np.empty(f.size)
    it = C.c_int64(0)
    res = C.c_double(0.0)
    conv = C.c_int(0)
    m = C.c_int(0)
    _check_ref(ref().ref_solve_truncated(dim, n, K, horizon_kind, delta0, coeff, _p(f), tol, max_iter,
                                         int(use_dense), _p(u), C.byref(it), C.byref(res), C.byref(conv),
                                         C.byref(m)))
    return u, it.value, res.value, bool(conv.value), m.value


def ref_dense_direct_solve(a, rhs):
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    x = np.empty(rhs.size)
    _check_ref(ref().ref_dense_direct_solve(rhs.size, _p(a), _p(rhs), _p(x)))
    return x


def ref_decompose(dim, n, center, radius, cap=1 << 20):
    """decompose_region: (levels, indices, recur_calls)."""
    c = np.zeros(3)
    c[:dim] = center
    lv = np.zeros(cap, dtype=np.int32)
    ix = np.zeros(cap, dtype=np.int64)
    npn, rc = C.c_int64(0), C.c_int64(0)
    _check_ref(ref().ref_decompose(dim, n, _p(c), radius, cap, lv.ctypes.data_as(C.POINTER(C.c_int)),
                                   ix.ctypes.data_as(_ip), C.byref(npn), C.byref(rc)))
    k = min(npn.value, cap)
    return lv[:k].copy(), ix[:k].copy(), rc.value


def ref_count_recur_calls(dim, n, radii):
    radii = np.ascontiguousarray(radii, dtype=np.float64)
    t = C.c_int64(0)
    _check_ref(ref().ref_count_recur_calls(dim, n, _p(radii), C.byref(t)))
    return t.value


def ref_moments(dim, n, K, u):
    u = np.ascontiguousarray(u, dtype=np.float64)
    L = int(round(np.log2(n)))
    nm = 2 * K + 1 if dim == 1 else 1
    size = sum((1 << (dim * l)) * nm for l in range(L + 1))
    out = np.empty(size)
    adds = C.c_int64(0)
    _check_ref(ref().ref_moments(dim, n, K, _p(u), _p(out), C.byref(adds)))
    return out, adds.value
