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


WORKLOADS = {"cfg0": cfg0, "cfg1": cfg1}
