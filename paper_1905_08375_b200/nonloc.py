"""Python mirror of the reference's operator API, backed by the B200 C-ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/nonloc/{geometry,kernel,operators}.hpp so that the
parity tests read like the reference's own tests:

  Grid.make                      geometry.hpp:18-26   (ValueError <- std::invalid_argument)
  RadialProfile.*, HorizonField  kernel.hpp:43-89
  KernelSpec                     kernel.hpp:94-108
  TruncatedOperator              operators.hpp:28-54  (ctor = Step 1, apply = Steps 2+3)
  apply_truncated_dense          operators.hpp:58-62
  apply_smooth_dense             operators.hpp:66-70
  apply_full_dense               operators.hpp:73-75
  apply_split                    operators.hpp:82-96
  match_polynomial, split        kernel.hpp:63-66
  ball_volume                    operators.hpp:22

Every apply runs on the GPU through include/nlgpu.h; there is no CPU path.
The BASELINE kernels the reference cannot express (fractional |r|^-alpha,
per-node delta / C / kappa arrays, zero collar, peridynamics) are exposed by
`NonlocalOperator` below.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, Optional, Sequence

import numpy as np

from . import _capi as A


class InclusionRule(IntEnum):
    Leaf = A.LEAF
    Point = A.POINT


class ApplyForm(IntEnum):
    Mass = A.MASS
    Difference = A.DIFFERENCE


class Exterior(IntEnum):
    Clip = A.CLIP
    Collar = A.COLLAR


class ProfileFamily(IntEnum):
    InverseS = 0
    ConicalInverseS = 1
    Regularized = 2
    PolynomialTruncated = 3


class HorizonKind(IntEnum):
    Constant = 0
    GaussianBump = 1


class SymmetryClass(IntEnum):
    NonDivergence = 0
    Divergence = 1


def _is_pow2(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


@dataclass(frozen=True)
class Grid:
    """Cell-centred grid on [0,1]^dim, node k at (k+1/2)h (geometry.hpp:16-26)."""
    dim: int = 1
    n: int = 2
    h: float = 0.5
    total: int = 2

    @staticmethod
    def make(dim: int, n: int, *, any_n: bool = False) -> "Grid":
        # geometry.cpp:11-24; any_n lifts the power-of-two restriction (SURVEY ledger L7)
        if dim < 1 or dim > 3:
            raise ValueError("grid dimension must be 1, 2 or 3")
        if n < 2 or (not any_n and not _is_pow2(n)):
            raise ValueError(f"grid n must be a power of two >= 2, got {n}")
        return Grid(dim, n, 1.0 / n, n ** dim)

    def levels(self) -> int:
        return int(round(math.log2(self.n)))


def match_polynomial(K: int, c: float = 1.0) -> np.ndarray:
    """p^{2K} coefficients for gamma = c/s (kernel.cpp:184-207)."""
    out = np.empty(K + 1)
    A.check(A.lib().nlg_match_polynomial(K, c, A.dptr(out)))
    return out


@dataclass
class SplitKernel:
    """gamma = kappa + p chi (kernel.hpp:29-41); tail per kernel.cpp:209-245."""
    scale: float
    order: int
    poly: np.ndarray
    tail: np.ndarray


def split(profile: "RadialProfile", K: int) -> SplitKernel:
    if profile.family != ProfileFamily.InverseS:
        raise ValueError("match_polynomial requires the InverseS profile")
    poly = np.empty(K + 1)
    tail = np.empty(K + 2)
    nt = C.c_int(0)
    A.check(A.lib().nlg_split(K, profile.c, A.dptr(poly), A.dptr(tail), C.byref(nt)))
    return SplitKernel(profile.c, K, poly, tail[: nt.value].copy())


@dataclass
class RadialProfile:
    family: ProfileFamily = ProfileFamily.InverseS
    c: float = 1.0
    order: int = 0
    poly: Optional[np.ndarray] = None
    split_data: Optional[SplitKernel] = None

    @staticmethod
    def inverse_s(c: float = 1.0) -> "RadialProfile":
        return RadialProfile(ProfileFamily.InverseS, c)

    @staticmethod
    def conical(c: float = 1.0) -> "RadialProfile":
        return RadialProfile(ProfileFamily.ConicalInverseS, c)

    @staticmethod
    def regularized(k: int, c: float = 1.0) -> "RadialProfile":
        return RadialProfile(ProfileFamily.Regularized, c, k,
                             split_data=split(RadialProfile.inverse_s(c), k))

    @staticmethod
    def truncated_polynomial(K: int, c: float = 1.0) -> "RadialProfile":
        return RadialProfile(ProfileFamily.PolynomialTruncated, c, K, poly=match_polynomial(K, c))

    def singular_at_origin(self) -> bool:
        return self.family != ProfileFamily.PolynomialTruncated


@dataclass
class HorizonField:
    kind: HorizonKind = HorizonKind.Constant
    delta0: float = 0.25

    def __call__(self, x0: float) -> float:
        # kernel.cpp:255-259 (math.exp is the C library exp the reference calls)
        if self.kind == HorizonKind.Constant:
            return self.delta0
        d = x0 - 0.5
        return self.delta0 * (1.0 + math.exp(-20.0 * d * d))

    def max_radius(self) -> float:
        return self.delta0 if self.kind == HorizonKind.Constant else 2.0 * self.delta0

    def nodes(self, grid: Grid) -> Optional[np.ndarray]:
        """delta at every node (axis-0 coordinate), or None when constant."""
        if self.kind == HorizonKind.Constant:
            return None
        col = np.array([self((k + 0.5) * grid.h) for k in range(grid.n)])
        return np.repeat(col, grid.n ** (grid.dim - 1))


@dataclass
class KernelSpec:
    dim: int = 1
    profile: RadialProfile = field(default_factory=RadialProfile)
    horizon: HorizonField = field(default_factory=HorizonField)
    symmetry: SymmetryClass = SymmetryClass.NonDivergence
    coefficient_value: float = 1.0
    # Arbitrary std::function coefficients cannot run on the GPU; a per-node
    # C(x) array is the supported form (SURVEY §8(b) ownership notes).
    coefficient_fn: Optional[Callable] = None
    coefficient_nodes: Optional[np.ndarray] = None


def ball_volume(dim: int, r: float) -> float:
    if dim == 1:
        return 2.0 * r
    if dim == 2:
        return math.pi * r * r
    if dim == 3:
        return 4.0 / 3.0 * math.pi * r * r * r
    raise ValueError("ball_volume: dim must be 1, 2 or 3")


# ---------------------------------------------------------------------------
# Plan: one nlg_plan
# ---------------------------------------------------------------------------

class Plan:
    """Owns one native plan (device buffers + stream). Arrays are copied in."""

    def __init__(self, *, dim, n, family, route=A.ROUTE_FULL, poly=None, tail=None, order=0,
                 c=1.0, alpha=1.0, rule=A.POINT, form=A.DIFFERENCE, exterior=A.CLIP,
                 divergence=False, delta=None, delta0=0.0, reach=0.0, coeff=None, coeff0=1.0,
                 kappa=None, row_begin=0, row_end=0, device=0):
        keep = []

        def arr(a):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(a)
            return a

        poly, tail, delta, coeff, kappa = map(arr, (poly, tail, delta, coeff, kappa))
        self.dim, self.n, self.family = dim, n, family
        self.components = dim if family == A.PERIDYNAMIC else 1
        self.desc = A.Desc(dim, n, family, route, A.dptr(poly), 0 if poly is None else len(poly),
                           A.dptr(tail), 0 if tail is None else len(tail), order, c, alpha, rule,
                           form, exterior, int(divergence), A.dptr(delta), delta0, reach,
                           A.dptr(coeff), coeff0, A.dptr(kappa), row_begin, row_end, device)
        h = C.c_void_p()
        A.check(A.lib().nlg_plan_create(C.byref(self.desc), C.byref(h)))
        self._h = h
        info = A.Info()
        A.check(A.lib().nlg_plan_info(self._h, C.byref(info)))
        self.info = info
        self.n_in, self.n_out = info.n_in, info.n_out

    def close(self):
        if getattr(self, "_h", None):
            A.lib().nlg_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _u(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
        if u.size != self.components * self.n_in:
            raise ValueError("u size does not match grid")
        return u

    def apply_fast(self, u) -> np.ndarray:
        u = self._u(u)
        out = np.empty(self.components * self.n_out)
        A.check(A.lib().nlg_apply_fast(self._h, A.dptr(u), A.dptr(out)))
        return out

    def apply_direct(self, u):
        u = self._u(u)
        out = np.empty(self.components * self.n_out)
        pairs = C.c_int64(0)
        A.check(A.lib().nlg_apply_direct(self._h, A.dptr(u), A.dptr(out), C.byref(pairs)))
        return out, pairs.value

    def apply_direct_at(self, u, targets, return_pairs: bool = False):
        """Direct sum at the given output nodes; with return_pairs, also the
        number of pairs summed (the reference's pair_count semantics)."""
        u = self._u(u)
        t = np.ascontiguousarray(targets, dtype=np.int64)
        out = np.empty(self.components * len(t))
        pairs = C.c_int64(0)
        A.check(A.lib().nlg_apply_direct_at(self._h, A.dptr(u), t.ctypes.data_as(A._ip), len(t),
                                            A.dptr(out), C.byref(pairs)))
        return (out, pairs.value) if return_pairs else out

    def apply_fast_dev(self, u_ptr: int, out_ptr: int, stream: int = 0) -> None:
        A.check(A.lib().nlg_apply_fast_dev(self._h, C.c_void_p(u_ptr), C.c_void_p(out_ptr),
                                           C.c_void_p(stream)))

    def apply_fast_dev_begin(self, u_ptr: int, out_ptr: int, stream: int = 0) -> None:
        """The halo-independent part of a sharded fast apply (nlg_apply_fast_dev_begin)."""
        A.check(A.lib().nlg_apply_fast_dev_begin(self._h, C.c_void_p(u_ptr), C.c_void_p(out_ptr),
                                                 C.c_void_p(stream)))

    def apply_fast_dev_end(self, u_ptr: int, out_ptr: int, stream: int = 0) -> None:
        A.check(A.lib().nlg_apply_fast_dev_end(self._h, C.c_void_p(u_ptr), C.c_void_p(out_ptr),
                                               C.c_void_p(stream)))

    def apply_fast_host_ptr(self, u_ptr: int, out_ptr: int) -> None:
        """nlg_apply_fast on raw host pointers (pinned buffers: the chunked
        H2D / apply / D2H pipeline overlaps its copies)."""
        A.check(A.lib().nlg_apply_fast(self._h, C.cast(u_ptr, A._dp), C.cast(out_ptr, A._dp)))

    def apply_direct_dev(self, u_ptr: int, out_ptr: int, pairs_ptr: int = 0, stream: int = 0) -> None:
        A.check(A.lib().nlg_apply_direct_dev(self._h, C.c_void_p(u_ptr), C.c_void_p(out_ptr),
                                             C.c_void_p(pairs_ptr or None), C.c_void_p(stream)))

    def apply_transpose(self, v) -> np.ndarray:
        """out = A^T v for the direct operator A (apply_direct)."""
        v = self._u(v)
        out = np.empty(self.n_out)
        A.check(A.lib().nlg_apply_transpose(self._h, A.dptr(v), A.dptr(out)))
        return out

    def assemble_dense(self) -> np.ndarray:
        """Dense row-major N x N matrix of the direct operator (unsharded plans)."""
        a = np.empty(self.n_out * self.n_out)
        A.check(A.lib().nlg_assemble_dense(self._h, A.dptr(a)))
        return a

    def solve_dirichlet(self, f, tol: float, max_iter: int, method: int = A.SOLVE_CG,
                        direct: bool = False) -> "SolveReport":
        """Device-resident CG / CGNR on A u = f with A = -L (this plan's fast
        apply, or its direct apply with direct=True)."""
        f = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
        if f.size != self.n_out:
            raise ValueError("f size does not match grid")
        u = np.empty(self.n_out)
        rep = A.SolveReport()
        A.check(A.lib().nlg_solve_dirichlet(self._h, A.dptr(f), tol, int(max_iter),
                                            int(method) | (A.SOLVE_DIRECT if direct else 0), A.dptr(u),
                                            C.byref(rep)))
        return SolveReport(SolveMethod(rep.method), rep.iterations, rep.final_residual, bool(rep.converged), u)

    def set_profiling(self, on: bool = True) -> None:
        A.check(A.lib().nlg_set_profiling(self._h, int(on)))

    def stage_times(self) -> dict:
        ms = np.zeros(len(A.STAGES))
        ln = np.zeros(len(A.STAGES), dtype=np.int64)
        n = C.c_int(0)
        A.check(A.lib().nlg_stage_times(self._h, A.dptr(ms), ln.ctypes.data_as(A._ip), C.byref(n)))
        return {A.STAGES[k]: (float(ms[k]), int(ln[k])) for k in range(n.value) if ln[k]}

    def launch_count(self) -> int:
        v = C.c_int64(0)
        A.check(A.lib().nlg_launch_count(self._h, C.byref(v)))
        return v.value

    def counters(self):
        p, f = C.c_int64(0), C.c_int64(0)
        A.check(A.lib().nlg_counters(self._h, C.byref(p), C.byref(f)))
        return p.value, f.value


def halo_rows(*, dim, n, family, delta_max, route=A.ROUTE_FULL, rule=A.POINT, form=A.DIFFERENCE,
              reach=0.0, poly=(1.0,), tail=(1.0,)) -> int:
    p = np.ascontiguousarray(poly, dtype=np.float64)
    t = np.ascontiguousarray(tail, dtype=np.float64)
    d = A.Desc(dim, n, family, route, A.dptr(p), len(p), A.dptr(t), len(t), 0, 1.0, 1.0, rule, form,
               0, 0, None, delta_max, reach, None, 1.0, None, 0, 0, 0)
    out = C.c_int64(0)
    A.check(A.lib().nlg_halo_rows(C.byref(d), delta_max, C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# reference-API mirror
# ---------------------------------------------------------------------------

def _check_u(grid: Grid, u) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
    if u.size != grid.total:
        raise ValueError("u size does not match grid")
    return u


def _coeff(spec: KernelSpec):
    if spec.coefficient_fn is not None:
        raise ValueError("coefficient_fn cannot run on the GPU; pass coefficient_nodes (C(x_i))")
    return spec.coefficient_nodes, spec.coefficient_value


def _profile_args(profile: RadialProfile):
    if profile.family == ProfileFamily.InverseS:
        return dict(family=A.INVERSE_S, c=profile.c)
    if profile.family == ProfileFamily.ConicalInverseS:
        return dict(family=A.CONICAL, c=profile.c)
    if profile.family == ProfileFamily.Regularized:
        sk = profile.split_data
        return dict(family=A.KAPPA, c=sk.scale, poly=sk.poly, tail=sk.tail, order=sk.order)
    return dict(family=A.TRUNCATED, c=profile.c, poly=profile.poly)


def _require_truncated(spec: KernelSpec):
    if spec.profile.family != ProfileFamily.PolynomialTruncated:
        raise ValueError("operation requires a PolynomialTruncated profile")


class TruncatedOperator:
    """Fast truncated operator (operators.hpp:28-54). The constructor is Step 1
    (plan creation: delta/C arrays to HBM, scan buffers); apply() is Steps 2+3
    on the GPU. K = 0 (any d) runs the span-prefix-sum kernels; K > 0 (1-D)
    runs the tiled polynomial quadrature (the raw-moment fast path is
    ill-conditioned, SURVEY ledger L4)."""

    def __init__(self, spec: KernelSpec, grid: Grid, device: int = 0):
        _require_truncated(spec)
        if spec.symmetry != SymmetryClass.NonDivergence:
            raise ValueError("the fast path is defined for the non-divergence form")
        K = spec.profile.order
        if grid.dim >= 2 and K != 0:
            raise ValueError("K > 0 is supported in 1d only")
        if grid.dim == 1 and K > 3:
            raise ValueError("K <= 3 in 1d")
        if not _is_pow2(grid.n):
            raise ValueError("tree requires n to be a power of two")
        self._spec, self._grid = spec, grid
        cn, cv = _coeff(spec)
        self._plan = Plan(dim=grid.dim, n=grid.n, family=A.TRUNCATED, route=A.ROUTE_TRUNCATED,
                          poly=spec.profile.poly, rule=A.LEAF, form=A.MASS,
                          delta=spec.horizon.nodes(grid), delta0=spec.horizon.delta0, coeff=cn,
                          coeff0=cv, device=device)
        self._applies = 0

    def apply(self, u) -> np.ndarray:
        u = _check_u(self._grid, u)
        self._applies += 1
        return self._plan.apply_fast(u)

    # -- Step-1 instruments (operators.hpp:35-42), computed lazily on the host --
    def _radii(self) -> np.ndarray:
        d = self._spec.horizon.nodes(self._grid)
        return np.full(self._grid.total, self._spec.horizon.delta0) if d is None else d

    def _tree_totals(self):
        if getattr(self, "_totals", None) is None:
            self._totals = count_tree(self._grid, self._radii())
        return self._totals

    def tree(self) -> "Tree":
        return build_tree(self._grid)

    def decompositions(self) -> list:
        """Per-node Algorithm-1 panel lists (host; O(N x panels) memory, as the reference)."""
        t = self.tree()
        r = self._radii()
        return [decompose_region(t, node_position(self._grid, i), float(r[i])) for i in range(self._grid.total)]

    def recur_calls(self) -> int:
        return self._tree_totals()[0]

    def step2_ops(self) -> int:
        nm = 2 * self._spec.profile.order + 1 if self._grid.dim == 1 else 1
        d, L = self._grid.dim, self._grid.levels()
        return self._applies * sum((1 << (d * l)) * (1 << d) * nm for l in range(L))

    def step3_ops(self) -> int:
        nm = 2 * self._spec.profile.order + 1 if self._grid.dim == 1 else 1
        return self._applies * self._tree_totals()[1] * nm

    def reset_counters(self) -> None:
        self._applies = 0

    def solve_dirichlet(self, f, tol: float, max_iter: int, method: Optional["SolveMethod"] = None) -> "SolveReport":
        """solve_dirichlet(-L, f) with the vectors resident on the GPU: CG for a
        symmetric operator (choose_method), CGNR with the GPU transpose apply
        otherwise (the reference assembles the dense matrix for this,
        tools/nonloc_main.cpp:200-219)."""
        m = choose_method(self._spec) if method is None else method
        return self._plan.solve_dirichlet(f, tol, max_iter, int(m))

    def spec(self):
        return self._spec

    def grid(self):
        return self._grid

    def fast_method(self) -> int:
        return self._plan.info.fast_method

    def applies(self) -> int:
        return self._applies


def apply_truncated_dense(spec: KernelSpec, grid: Grid, rule: InclusionRule, u,
                          form: ApplyForm = ApplyForm.Mass, pair_count: Optional[list] = None,
                          device: int = 0) -> np.ndarray:
    _require_truncated(spec)
    u = _check_u(grid, u)
    cn, cv = _coeff(spec)
    p = Plan(dim=grid.dim, n=grid.n, family=A.TRUNCATED, route=A.ROUTE_TRUNCATED,
             poly=spec.profile.poly, rule=int(rule), form=int(form), delta=spec.horizon.nodes(grid),
             delta0=spec.horizon.delta0, coeff=cn, coeff0=cv, device=device)
    out, pairs = p.apply_direct(u)
    if pair_count is not None:
        pair_count.append(pairs)
    return out


def apply_smooth_dense(sk: SplitKernel, spec: KernelSpec, grid: Grid, u,
                       pair_count: Optional[list] = None, device: int = 0) -> np.ndarray:
    u = _check_u(grid, u)
    cn, cv = _coeff(spec)
    p = Plan(dim=grid.dim, n=grid.n, family=A.KAPPA, route=A.ROUTE_SMOOTH, c=sk.scale, poly=sk.poly,
             tail=sk.tail, order=sk.order, rule=A.POINT, form=A.DIFFERENCE,
             delta=spec.horizon.nodes(grid), delta0=spec.horizon.delta0, coeff=cn, coeff0=cv,
             device=device)
    out, pairs = p.apply_direct(u)
    if pair_count is not None:
        pair_count.append(pairs)
    return out


def apply_full_dense(spec: KernelSpec, grid: Grid, u, pair_count: Optional[list] = None,
                     device: int = 0) -> np.ndarray:
    u = _check_u(grid, u)
    cn, cv = _coeff(spec)
    p = Plan(dim=grid.dim, n=grid.n, route=A.ROUTE_FULL, rule=A.POINT, form=A.DIFFERENCE,
             divergence=spec.symmetry == SymmetryClass.Divergence, delta=spec.horizon.nodes(grid),
             delta0=spec.horizon.delta0, reach=spec.horizon.max_radius(), coeff=cn, coeff0=cv,
             device=device, **_profile_args(spec.profile))
    out, pairs = p.apply_direct(u)
    if pair_count is not None:
        pair_count.append(pairs)
    return out


class SmoothBackend(IntEnum):
    Dense = 0
    Hodlr = 1


class TruncatedPath(IntEnum):
    FastLeafMass = 0
    DensePointDifference = 1


@dataclass
class SplitApplyOptions:
    backend: SmoothBackend = SmoothBackend.Dense
    truncated: TruncatedPath = TruncatedPath.FastLeafMass
    epsilon: float = 1e-8


def apply_split(spec: KernelSpec, grid: Grid, K: int, u,
                options: SplitApplyOptions = SplitApplyOptions(), device: int = 0) -> np.ndarray:
    """operators.cpp:305-337. The HODLR backend is out of scope."""
    if spec.profile.family != ProfileFamily.InverseS:
        raise ValueError("apply_split expects the InverseS profile")
    if options.backend != SmoothBackend.Dense:
        raise ValueError("HODLR smooth backend is out of scope for the GPU build")
    sk = split(spec.profile, K)
    out = apply_smooth_dense(sk, spec, grid, u, device=device)
    tspec = KernelSpec(spec.dim, RadialProfile.truncated_polynomial(K, spec.profile.c), spec.horizon,
                       spec.symmetry, spec.coefficient_value, spec.coefficient_fn,
                       spec.coefficient_nodes)
    if options.truncated == TruncatedPath.FastLeafMass:
        tpart = TruncatedOperator(tspec, grid, device=device).apply(u)
    else:
        tpart = apply_truncated_dense(tspec, grid, InclusionRule.Point, u, ApplyForm.Difference,
                                      device=device)
    return out + tpart


# ---------------------------------------------------------------------------
# BASELINE operators (no reference equivalent)
# ---------------------------------------------------------------------------

def fractional_cdelta(dim: int, s: float, delta):
    """C_delta with int_{B_delta} |z|^2 C_delta |z|^{-(d+2s)} dz = 1 (SURVEY ledger L6):
    C_delta = (2-2s) / (|S^{d-1}| delta^{2-2s}), |S^0|=2, |S^1|=2 pi, |S^2|=4 pi."""
    area = {1: 2.0, 2: 2.0 * math.pi, 3: 4.0 * math.pi}[dim]
    return (2.0 - 2.0 * s) / (area * np.power(delta, 2.0 - 2.0 * s))


class NonlocalOperator:
    """L u(x) = h^d sum_{y != x, |y-x| < delta(x)} omega(x,y) (u(y) - u(x)) on the
    uniform grid, omega = C(x) (kappa(x)+kappa(y))/2 |y-x|^-alpha (fractional)
    or the bond-based peridynamic operator. apply() is the fast path,
    apply_direct() the O(N (delta/h)^d) direct quadrature (in-repo oracle)."""

    def __init__(self, dim: int, n: int, *, kernel: str = "fractional", alpha: float = 1.0,
                 delta=None, delta0: float = 0.0, coeff=None, coeff0: float = 1.0, kappa=None,
                 exterior: Exterior = Exterior.Clip, row_begin: int = 0, row_end: int = 0,
                 reach: float = 0.0, device: int = 0):
        fam = A.FRACTIONAL if kernel == "fractional" else A.PERIDYNAMIC
        self.grid = Grid.make(dim, n, any_n=True)
        self.plan = Plan(dim=dim, n=n, family=fam, alpha=alpha, rule=A.POINT, form=A.DIFFERENCE,
                         exterior=int(exterior), delta=delta, delta0=delta0, coeff=coeff,
                         coeff0=coeff0, kappa=kappa, reach=reach, row_begin=row_begin,
                         row_end=row_end, device=device)

    @property
    def info(self):
        return self.plan.info

    def apply(self, u) -> np.ndarray:
        return self.plan.apply_fast(u)

    def apply_direct(self, u):
        return self.plan.apply_direct(u)

    def apply_direct_at(self, u, targets, return_pairs: bool = False):
        return self.plan.apply_direct_at(u, targets, return_pairs)


class Group:
    """Multi-GPU operator (nlg_group_*, csrc/group.cu): the grid split into
    axis-0 slabs over `devices`, one sharded plan per device, u's halo rows
    exchanged device to device by NCCL (a repeated device ordinal: peer
    copies), overlapped with the halo-independent part of each apply.
    Arguments as Plan, over the whole grid."""

    def __init__(self, devices, *, dim, n, family, route=A.ROUTE_FULL, poly=None, alpha=1.0, rule=A.POINT,
                 form=A.DIFFERENCE, exterior=A.CLIP, delta=None, delta0=0.0, coeff=None, coeff0=1.0, kappa=None):
        keep = []

        def arr(a):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(a)
            return a

        poly, delta, coeff, kappa = map(arr, (poly, delta, coeff, kappa))
        self.dim, self.n = dim, n
        self.components = dim if family == A.PERIDYNAMIC else 1
        desc = A.Desc(dim, n, family, route, A.dptr(poly), 0 if poly is None else len(poly), None, 0, 0, 1.0,
                      alpha, rule, form, int(exterior), 0, A.dptr(delta), delta0, 0.0, A.dptr(coeff), coeff0,
                      A.dptr(kappa), 0, 0, 0)
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        A.check(A.lib().nlg_group_create(C.byref(desc), len(devices), devs, C.byref(h)), group=True)
        self._h = h
        nd, nc = C.c_int(0), C.c_int(0)
        rb = np.zeros(len(devices), dtype=np.int64)
        re = np.zeros(len(devices), dtype=np.int64)
        nin = np.zeros(len(devices), dtype=np.int64)
        A.check(A.lib().nlg_group_info(self._h, C.byref(nd), C.byref(nc), rb.ctypes.data_as(A._ip),
                                       re.ctypes.data_as(A._ip), nin.ctypes.data_as(A._ip)), group=True)
        self.ndev, self.nccl = nd.value, bool(nc.value)
        self.row_begin, self.row_end, self.n_in = rb, re, nin

    def apply(self, u) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
        if u.size != self.components * self.n ** self.dim:
            raise ValueError("u size does not match grid")
        out = np.empty_like(u)
        A.check(A.lib().nlg_group_apply_fast(self._h, A.dptr(u), A.dptr(out)), group=True)
        return out

    def apply_dev(self, u_ptrs, out_ptrs) -> None:
        up = (C.c_void_p * self.ndev)(*u_ptrs)
        op = (C.c_void_p * self.ndev)(*out_ptrs)
        A.check(A.lib().nlg_group_apply_fast_dev(self._h, up, op), group=True)

    def close(self):
        if getattr(self, "_h", None):
            A.lib().nlg_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Krylov consumer (reference include/nonloc/solve.hpp, src/solve.cpp)
# ---------------------------------------------------------------------------

class SolveMethod(IntEnum):
    CG = 0
    CGNR = 1


@dataclass
class SolveReport:
    method: SolveMethod = SolveMethod.CG
    iterations: int = 0
    final_residual: float = 0.0        # ||f - A u||_2 / ||f||_2
    converged: bool = False
    solution: Optional[np.ndarray] = None


def choose_method(spec: KernelSpec) -> SolveMethod:
    """CG when the configuration yields a symmetric matrix (solve.cpp:110-114)."""
    symmetric = spec.horizon.kind == HorizonKind.Constant and spec.coefficient_fn is None
    return SolveMethod.CG if symmetric else SolveMethod.CGNR


def solve_dirichlet(apply, f, tol: float, max_iter: int, method: SolveMethod = SolveMethod.CG,
                    apply_transpose=None) -> SolveReport:
    """Matrix-free Krylov solve of A u = f for an arbitrary `apply` callable
    (the reference's ApplyFn, solve.cpp:32-108), same recurrences and stopping
    rules. For a GPU operator prefer TruncatedOperator.solve_dirichlet /
    Plan.solve_dirichlet, which keep every vector in HBM."""
    f = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
    n = f.size
    rep = SolveReport(method=method, solution=np.zeros(n))
    fnorm = float(np.sqrt(np.dot(f, f)))
    if fnorm == 0.0:
        rep.converged = True
        return rep
    if method == SolveMethod.CGNR and apply_transpose is None:
        raise ValueError("CGNR needs the transpose application")

    def checked(v):
        v = np.asarray(v, dtype=np.float64)
        if not np.all(np.isfinite(v)):
            raise A.NonlocError("operator produced a non-finite value")
        return v

    u = rep.solution
    r = f.copy()
    if method == SolveMethod.CG:
        p = r.copy()
        rr = float(np.dot(r, r))
        for it in range(max_iter):
            if np.sqrt(rr) / fnorm <= tol:
                break
            ap = checked(apply(p))
            pap = float(np.dot(p, ap))
            if pap == 0.0:
                break
            alpha = rr / pap
            u += alpha * p
            r -= alpha * ap
            rr_next = float(np.dot(r, r))
            beta = rr_next / rr
            rr = rr_next
            p = r + beta * p
            rep.iterations = it + 1
    else:
        z = np.asarray(apply_transpose(r), dtype=np.float64)
        p = z.copy()
        zz = float(np.dot(z, z))
        for it in range(max_iter):
            if np.sqrt(np.dot(r, r)) / fnorm <= tol:
                break
            ap = checked(apply(p))
            denom = float(np.dot(ap, ap))
            if denom == 0.0:
                break
            alpha = zz / denom
            u += alpha * p
            r -= alpha * ap
            z = checked(apply_transpose(r))
            zz_next = float(np.dot(z, z))
            beta = zz_next / zz
            zz = zz_next
            p = z + beta * p
            rep.iterations = it + 1
    au = np.asarray(apply(u), dtype=np.float64)
    rep.final_residual = float(np.sqrt(np.sum((f - au) ** 2)) / fnorm)
    rep.converged = rep.final_residual <= tol
    return rep


def dense_direct_solve(a_rowmajor, rhs) -> np.ndarray:
    """Partial-pivot LU solve of the row-major n x n system (oracle path,
    solve.cpp:116-127)."""
    rhs = np.asarray(rhs, dtype=np.float64).reshape(-1)
    n = rhs.size
    a = np.asarray(a_rowmajor, dtype=np.float64).reshape(-1)
    if a.size != n * n:
        raise ValueError("dense_direct_solve: shape mismatch")
    return np.linalg.solve(a.reshape(n, n), rhs)


def assemble_dense_matrix(spec: KernelSpec, grid: Grid, rule: InclusionRule, form: ApplyForm,
                          device: int = 0) -> np.ndarray:
    """Dense row-major matrix of the direct operator (operators.cpp:262-303),
    assembled on the GPU (one thread per row)."""
    if form == ApplyForm.Mass:
        _require_truncated(spec)
    cn, cv = _coeff(spec)
    if spec.profile.family == ProfileFamily.PolynomialTruncated:
        p = Plan(dim=grid.dim, n=grid.n, family=A.TRUNCATED, route=A.ROUTE_TRUNCATED,
                 poly=spec.profile.poly, rule=int(rule), form=int(form), delta=spec.horizon.nodes(grid),
                 delta0=spec.horizon.delta0, coeff=cn, coeff0=cv, device=device)
    else:
        p = Plan(dim=grid.dim, n=grid.n, route=A.ROUTE_FULL, rule=A.POINT, form=A.DIFFERENCE,
                 divergence=spec.symmetry == SymmetryClass.Divergence, delta=spec.horizon.nodes(grid),
                 delta0=spec.horizon.delta0, reach=spec.horizon.max_radius(), coeff=cn, coeff0=cv,
                 device=device, **_profile_args(spec.profile))
    return p.assemble_dense()


# ---------------------------------------------------------------------------
# Step-1 tree API (reference include/nonloc/tree.hpp), host side
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class PanelId:
    level: int
    index: int


@dataclass
class Tree:
    grid: Grid
    depth: int

    def panels_at(self, level: int) -> int:
        return 1 << (self.grid.dim * level)

    def _k(self, pid: PanelId):
        per = 1 << pid.level
        rest, k = pid.index, [0, 0, 0]
        for j in range(self.grid.dim - 1, -1, -1):
            k[j] = rest % per
            rest //= per
        return k

    def child(self, pid: PanelId, which: int) -> PanelId:
        per, k = 1 << pid.level, self._k(pid)
        f = 0
        for j in range(self.grid.dim):
            f = f * (2 * per) + (2 * k[j] + ((which >> j) & 1))
        return PanelId(pid.level + 1, f)

    def parent(self, pid: PanelId) -> PanelId:
        if pid.level == 0:
            raise ValueError("root has no parent")
        per, k = 1 << pid.level, self._k(pid)
        f = 0
        for j in range(self.grid.dim):
            f = f * (per // 2) + k[j] // 2
        return PanelId(pid.level - 1, f)

    def bounds(self, pid: PanelId):
        w = 1.0 / (1 << pid.level)
        k = self._k(pid)
        return ([k[j] * w for j in range(self.grid.dim)], [(k[j] + 1) * w for j in range(self.grid.dim)])

    def is_leaf(self, pid: PanelId) -> bool:
        return pid.level == self.depth


def build_tree(grid: Grid) -> Tree:
    if not _is_pow2(grid.n):
        raise ValueError("tree requires n to be a power of two")
    return Tree(grid, grid.levels())


def node_position(grid: Grid, i: int) -> np.ndarray:
    k, rest = [0, 0, 0], int(i)
    for j in range(grid.dim - 1, -1, -1):
        k[j] = rest % grid.n
        rest //= grid.n
    return np.array([(k[j] + 0.5) * grid.h for j in range(grid.dim)])


@dataclass
class Decomposition:
    center: np.ndarray
    radius: float
    panels: list
    recur_calls: int


def decompose_region(tree: Tree, center, radius: float) -> Decomposition:
    """Algorithm 1 panels (pre-order) covering B_r(center) at leaf resolution."""
    if radius <= 0.0:
        raise ValueError("radius must be positive")
    c = np.zeros(3)
    c[:tree.grid.dim] = np.asarray(center, dtype=np.float64).reshape(-1)[:tree.grid.dim]
    cap = 1 << 16
    while True:
        lv = np.zeros(cap, dtype=np.int32)
        ix = np.zeros(cap, dtype=np.int64)
        npn, rc = C.c_int64(0), C.c_int64(0)
        A.check(A.lib().nlg_tree_decompose(tree.grid.dim, tree.grid.n, A.dptr(c), radius, cap,
                                           lv.ctypes.data_as(C.POINTER(C.c_int)), ix.ctypes.data_as(A._ip),
                                           C.byref(npn), C.byref(rc)))
        if npn.value <= cap:
            break
        cap = npn.value
    panels = [PanelId(int(lv[k]), int(ix[k])) for k in range(npn.value)]
    return Decomposition(c[:tree.grid.dim].copy(), radius, panels, rc.value)


def count_tree(grid: Grid, radii) -> tuple:
    """(recur calls, panels) summed over every node's ball (host threads)."""
    r = np.ascontiguousarray(radii, dtype=np.float64)
    if r.size != grid.total:
        raise ValueError("radii size does not match grid")
    rc, pc = C.c_int64(0), C.c_int64(0)
    A.check(A.lib().nlg_tree_count(grid.dim, grid.n, A.dptr(r), C.byref(rc), C.byref(pc)))
    return rc.value, pc.value


def count_recur_calls(tree: Tree, radii) -> int:
    return count_tree(tree.grid, radii)[0]


@dataclass
class MomentTable:
    num_moments: int
    levels: list

    def moment(self, pid: PanelId, m: int) -> float:
        return float(self.levels[pid.level][pid.index * self.num_moments + m])


def accumulate_moments(tree: Tree, u, K: int, add_count: Optional[list] = None) -> MomentTable:
    g = tree.grid
    u = _check_u(g, u)
    if K < 0 or (g.dim >= 2 and K != 0):
        raise ValueError("moments support K >= 0 in 1d, K = 0 in 2d/3d")
    nm = 2 * K + 1 if g.dim == 1 else 1
    sizes = [tree.panels_at(l) * nm for l in range(tree.depth + 1)]
    out = np.empty(sum(sizes))
    adds = C.c_int64(0)
    A.check(A.lib().nlg_tree_moments(g.dim, g.n, K, A.dptr(u), A.dptr(out), C.byref(adds)))
    if add_count is not None:
        add_count.append(adds.value)
    levels, o = [], 0
    for sz in sizes:
        levels.append(out[o:o + sz])
        o += sz
    return MomentTable(nm, levels)
