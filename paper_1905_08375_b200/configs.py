"""Seeded synthetic workloads for the BASELINE.json configs (no datasets exist
for this path). Every field is generated on the host with numpy's
PCG64 from a fixed seed and shipped as an array, so the GPU kernels and the CPU
oracle read bit-identical inputs.

Seeds (recorded in every bench line): u -> 1, kappa / c -> 2, delta -> 3,
inclusion geometry -> 4 (SURVEY §8(d) suggestion).

C_delta follows SURVEY ledger L6:  int_{B_delta} |z|^2 C_delta |z|^{-(d+2s)} dz = 1.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .nonloc import fractional_cdelta


@dataclass
class Workload:
    name: str
    dim: int
    n: int
    kernel: str                      # "fractional" | "peridynamic"
    alpha: float
    s: float
    u: np.ndarray
    delta: Optional[np.ndarray] = None
    delta0: float = 0.0
    coeff: Optional[np.ndarray] = None
    coeff0: float = 1.0
    kappa: Optional[np.ndarray] = None
    exterior: int = 0               # 0 clip, 1 zero collar
    seeds: dict = field(default_factory=dict)
    algo_bytes: int = 16            # algorithmic HBM bytes per point
    # kernel == "truncated": the reference's own fast route, TruncatedOperator
    # (operators.cpp:102-167), polynomial profile of order K, Leaf rule, Mass form
    K: int = 0
    horizon_kind: int = 0           # 0 Constant, 1 GaussianBump (kernel.hpp:80-89)

    @property
    def N(self) -> int:
        return self.n ** self.dim

    def op_kwargs(self) -> dict:
        return dict(kernel=self.kernel, alpha=self.alpha, delta=self.delta, delta0=self.delta0,
                    coeff=self.coeff, coeff0=self.coeff0, kappa=self.kappa, exterior=self.exterior)

    def oracle_kwargs(self) -> dict:
        import oracle as O  # test infrastructure only (tests/, bench cpu leg)
        return dict(family=O.PERIDYNAMIC if self.kernel == "peridynamic" else O.FRACTIONAL,
                    alpha=self.alpha, delta=self.delta, delta0=self.delta0, coeff=self.coeff,
                    coeff0=self.coeff0, kappa=self.kappa, exterior=self.exterior,
                    peri=self.kernel == "peridynamic")

    def bytes_per_point(self) -> int:
        """Algorithmic HBM bytes per output point: every input field read once,
        the output written once; C_delta(x) is a function of
        delta(x) and is not counted as a field."""
        return self.algo_bytes


def _nodes(n: int) -> np.ndarray:
    return (np.arange(n) + 0.5) / n


def _u_1d(n: int, rng: np.random.Generator) -> np.ndarray:
    # u = sum_{k=1..16} a_k sin(2 pi k x), a_k ~ N(0, 1/k^2), + 1e-3 U(-1,1)
    x = _nodes(n)
    k = np.arange(1, 17)
    a = rng.standard_normal(16) / k
    u = np.zeros(n)
    for kk, aa in zip(k, a):
        u += aa * np.sin(2 * math.pi * kk * x)
    return u + 1e-3 * rng.uniform(-1.0, 1.0, n)


def _smooth_1d(n: int, modes: int, rng: np.random.Generator) -> np.ndarray:
    x = _nodes(n)
    g = np.zeros(n)
    for k in range(1, modes + 1):
        a, b = rng.standard_normal(2) / k
        g += a * np.cos(2 * math.pi * k * x) + b * np.sin(2 * math.pi * k * x)
    return g


def _lognormal_1d(n: int, rng: np.random.Generator, sigma: float = 0.5) -> np.ndarray:
    g = _smooth_1d(n, 32, rng)
    g = (g - g.mean()) / g.std() * sigma
    return np.exp(g)


def cfg0(n: int = 4096) -> Workload:
    """1-D, N=4096, delta=0.02, s=0.25, zero collar; fast and direct apply."""
    s, delta0 = 0.25, 0.02
    u = _u_1d(n, np.random.default_rng(1))
    return Workload("cfg0_1d_fractional_collar", 1, n, "fractional", 1 + 2 * s, s, u, delta0=delta0,
                    coeff0=float(fractional_cdelta(1, s, delta0)), exterior=1, seeds={"u": 1},
                    algo_bytes=16)


def cfg1(n: int = 1 << 22, exterior: int = 0) -> Workload:
    """1-D, N=2^22, delta(x)=0.005+0.01(1/2+1/2 sin 2 pi x), s=0.4,
    kappa-weighted (kappa = exp(g), 32 modes, sigma 0.5). Exterior: clip by
    default — the reference's own apply_full_dense convention
    (operators.cpp:36-38), so the compiled reference evaluates the identical
    operator; exterior=1 gives the zero collar (kappa_y := kappa_x outside)."""
    s = 0.4
    x = _nodes(n)
    delta = 0.005 + 0.01 * (0.5 + 0.5 * np.sin(2 * math.pi * x))
    u = _u_1d(n, np.random.default_rng(1))
    kappa = _lognormal_1d(n, np.random.default_rng(2))
    coeff = fractional_cdelta(1, s, delta)
    return Workload("cfg1_1d_kappa_variable_delta", 1, n, "fractional", 1 + 2 * s, s, u, delta=delta,
                    coeff=coeff, kappa=kappa, exterior=exterior, seeds={"u": 1, "kappa": 2},
                    algo_bytes=32)


# ---------------------------------------------------------------------------
# 2-D / 3-D workloads. Fields are sums of seeded Fourier modes evaluated with
# torch (on the GPU when one is present — 768^3 has 4.5e8 nodes), returned as
# numpy arrays so the plan and the oracle read identical inputs.
# ---------------------------------------------------------------------------

def _torch_dev():
    import torch
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


def _modes(rng, count, kmax, dim, decay=1.0):
    ks = rng.integers(-kmax, kmax + 1, size=(count, dim))
    ks[np.all(ks == 0, axis=1)] = 1
    amp = rng.standard_normal(count) / np.linalg.norm(ks, axis=1) ** decay
    ph = rng.uniform(0.0, 2 * math.pi, count)
    return ks, amp, ph


def _field(n, dim, ks, amp, ph):
    """sum_m amp_m sin(2 pi k_m . x + ph_m) on the cell centres, row-major."""
    import torch
    dev = _torch_dev()
    x = (torch.arange(n, device=dev, dtype=torch.float64) + 0.5) / n
    shape = [n] * dim
    out = torch.zeros(shape, device=dev, dtype=torch.float64)
    for k, a, p in zip(ks, amp, ph):
        arg = torch.full(shape, float(p), device=dev, dtype=torch.float64)
        for j in range(dim):
            view = [1] * dim
            view[j] = n
            arg = arg + (2 * math.pi * float(k[j])) * x.view(view)
        out += float(a) * torch.sin(arg)
    return out.reshape(-1).cpu().numpy()


def _noise(n_total, rng):
    return 1e-3 * rng.uniform(-1.0, 1.0, n_total)


def _lognormal(n, dim, rng, sigma=0.5, modes=32):
    ks, amp, ph = _modes(rng, modes, 4, dim)
    g = _field(n, dim, ks, amp, ph)
    return np.exp((g - g.mean()) / g.std() * sigma)


def cfg2(n: int = 4096) -> Workload:
    """2-D, 4096^2, delta(x) = h (8 + 4 sin(2 pi k.x + phi)) in [4h, 12h],
    s = 0.5 (|r|^-3), kappa lognormal (sigma 0.5), u = 64 modes + noise."""
    s, dim = 0.5, 2
    h = 1.0 / n
    rd = np.random.default_rng(3)
    k = rd.integers(1, 5, size=(1, dim))
    delta = h * (8.0 + 4.0 * _field(n, dim, k, np.ones(1), rd.uniform(0, 2 * math.pi, 1)))
    ru = np.random.default_rng(1)
    ks, amp, ph = _modes(ru, 64, 8, dim)
    u = _field(n, dim, ks, amp, ph) + _noise(n ** dim, ru)
    kappa = _lognormal(n, dim, np.random.default_rng(2))
    coeff = fractional_cdelta(dim, s, delta)
    return Workload("cfg2_2d_kappa_variable_delta", dim, n, "fractional", dim + 2 * s, s, u, delta=delta,
                    coeff=coeff, kappa=kappa, exterior=0, seeds={"u": 1, "kappa": 2, "delta": 3},
                    algo_bytes=32)


def cfg3(n: int = 4096) -> Workload:
    """2-D bond-based peridynamics, 4096^2, u in R^2 (SoA planes), circular
    inclusion (centre U([.3,.7]^2), radius U(.1,.25)); delta in [3h,5h] inside,
    [5h,8h] outside (smooth within each material); c_in = 10 c_out."""
    dim = 2
    h = 1.0 / n
    rg = np.random.default_rng(4)
    cen = rg.uniform(0.3, 0.7, 2)
    rad = rg.uniform(0.1, 0.25)
    x = (np.arange(n) + 0.5) / n
    inside = ((x[:, None] - cen[0]) ** 2 + (x[None, :] - cen[1]) ** 2 < rad * rad).reshape(-1)
    rd = np.random.default_rng(3)
    k = rd.integers(1, 5, size=(1, dim))
    wave = _field(n, dim, k, np.ones(1), rd.uniform(0, 2 * math.pi, 1))
    delta = np.where(inside, h * (4.0 + wave), h * (6.5 + 1.5 * wave))
    coeff = np.where(inside, 10.0, 1.0)
    ru = np.random.default_rng(1)
    comps = []
    for _ in range(2):
        ks, amp, ph = _modes(ru, 64, 8, dim)
        comps.append(_field(n, dim, ks, amp, ph))
    u = np.concatenate(comps)
    return Workload("cfg3_2d_peridynamics_inclusion", dim, n, "peridynamic", 1.0, 0.0, u, delta=delta,
                    coeff=coeff, exterior=0, seeds={"u": 1, "delta": 3, "inclusion": 4}, algo_bytes=48)


def cfg4(n: int = 768, variable: bool = False) -> Workload:
    """3-D, 768^3 (non power of two), delta = 6h (A) or h (6 + 2 sin(.)) in
    [4h, 8h] (B); s = 0.25 (|r|^-3.5), kappa lognormal, u = 128 modes."""
    s, dim = 0.25, 3
    h = 1.0 / n
    if variable:
        rd = np.random.default_rng(3)
        k = rd.integers(1, 4, size=(1, dim))
        delta = h * (6.0 + 2.0 * _field(n, dim, k, np.ones(1), rd.uniform(0, 2 * math.pi, 1)))
        coeff = fractional_cdelta(dim, s, delta)
        d0 = 0.0
        c0 = 1.0
    else:
        delta, d0 = None, 6.0 * h
        coeff, c0 = None, float(fractional_cdelta(dim, s, 6.0 * h))
    ru = np.random.default_rng(1)
    ks, amp, ph = _modes(ru, 128, 8, dim)
    u = _field(n, dim, ks, amp, ph)
    kappa = _lognormal(n, dim, np.random.default_rng(2))
    name = "cfg4B_3d_kappa_variable_delta" if variable else "cfg4A_3d_kappa_delta6h"
    return Workload(name, dim, n, "fractional", dim + 2 * s, s, u, delta=delta, delta0=d0, coeff=coeff,
                    coeff0=c0, kappa=kappa, exterior=0, seeds={"u": 1, "kappa": 2, "delta": 3},
                    algo_bytes=32 if variable else 24)


def trunc1d(n: int = 1 << 22) -> Workload:
    """The reference's own fast route on the cfg1 grid:
    TruncatedOperator, 1-D N=2^22, Gaussian-bump horizon delta0=0.005
    (delta in [0.005, 0.01]), K=0, C=1, Leaf rule, Mass form; u = 16 modes +
    noise (as cfg0/cfg1). The reference arm times TruncatedOperator::apply
    (Steps 2+3, bench.cpp:47-49) on the same grid."""
    u = _u_1d(n, np.random.default_rng(1))
    return Workload("trunc1d_K0_bump_n4194304", 1, n, "truncated", 0.0, 0.0, u, delta0=0.005,
                    coeff0=1.0, seeds={"u": 1}, algo_bytes=16, K=0, horizon_kind=1)


def trunc2d(n: int = 1024) -> Workload:
    """TruncatedOperator in 2-D, 1024^2, constant delta = 8h, K=0."""
    ru = np.random.default_rng(1)
    ks, amp, ph = _modes(ru, 64, 8, 2)
    u = _field(n, 2, ks, amp, ph) + _noise(n * n, ru)
    return Workload("trunc2d_K0_delta8h_n1024", 2, n, "truncated", 0.0, 0.0, u, delta0=8.0 / n,
                    coeff0=1.0, seeds={"u": 1}, algo_bytes=16, K=0, horizon_kind=0)


WORKLOADS = {"cfg0": cfg0, "cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4,
             "cfg4b": lambda n=768: cfg4(n, variable=True), "trunc1d": trunc1d, "trunc2d": trunc2d}
