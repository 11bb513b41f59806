"""B200-native nonlocal-operator apply (Tian & Engquist, arXiv 1905.08375).

The hot path is hand-written sm_100a CUDA behind the C-ABI in include/nlgpu.h
(paper_1905_08375_b200/_lib/libnlgpu.so). `nonloc` mirrors the reference's
C++ operator API; `slabs` shards a grid across ranks along axis 0.
"""
from . import _capi
from .nonloc import (ApplyForm, Exterior, Grid, HorizonField, HorizonKind, InclusionRule, KernelSpec,
                     NonlocalOperator, Plan, ProfileFamily, RadialProfile, SmoothBackend,
                     SplitApplyOptions, SplitKernel, SymmetryClass, TruncatedOperator, TruncatedPath,
                     apply_full_dense, apply_smooth_dense, apply_split, apply_truncated_dense,
                     ball_volume, fractional_cdelta, halo_rows, match_polynomial, split)

__all__ = [n for n in dir() if not n.startswith("_")]
