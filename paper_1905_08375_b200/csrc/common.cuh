// paper_1905_08375_b200/csrc/common.cuh — shared device helpers.
//
// The quadrature contract (which nodes enter a sum) must be reproduced
// bit-exactly (SURVEY.md §7 hard part 1). Every predicate below evaluates the
// same IEEE operations, in the same order, as the reference:
//   node_position   (k+1/2)h                       geometry.cpp:78-84
//   dist            sqrt(sum (y_j-x_j)^2)          operators.cpp:71-78
//   Leaf rule       cube_intersects_ball(leaf box) geometry.cpp:63-76, operators.cpp:44-51
// using the _rn intrinsics so nvcc cannot contract them into FMAs.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nlg {

constexpr int kMaxPoly = 8;   // p(s) coefficients (K <= 7)
constexpr int kMaxTail = 16;

// Kernel profile constants, passed by value to every kernel.
struct Profile {
  int family;
  int route;
  int npoly, ntail, order;
  double c, alpha;
  double poly[kMaxPoly];
  double tail[kMaxTail];
};

// Geometry of a (possibly sharded) grid: output rows [row_begin,row_end) of
// axis 0, input arrays cover rows [in_begin, in_end).
struct Geom {
  int dim;
  int64_t n;          // nodes per axis
  double h;           // 1/n
  double hd;          // h^d, same multiply order as hd_weight (operators.cpp:85-89)
  int64_t stride0;    // nodes per axis-0 row = n^{d-1}
  int64_t row_begin, row_end;  // output rows
  int64_t in_begin, in_end;    // input rows
};

// Relative half-width of the tie band around (delta/h)^2 in which integer
// |d|^2 classification defers to the reference's float predicate. The
// predicate's r2 carries a relative error up to ~7 eps n / |d| when h = 1/n is
// inexact (non-power-of-two n), so the band grows with n: 1e-12 + 8 eps n.
__host__ __device__ __forceinline__ double tie_band(double h) {
  return 1e-12 + 8.0 * 2.220446049250313e-16 / h;
}
__host__ __device__ __forceinline__ double tie_band_n(double inv_h) {
  return 1e-12 + 8.0 * 2.220446049250313e-16 * inv_h;
}

__device__ __forceinline__ double coord(int64_t k, double h) {
  return __dmul_rn(__dadd_rn(static_cast<double>(k), 0.5), h);
}

__device__ __forceinline__ double delta_power(int dim, double delta) {
  double p = __dmul_rn(delta, delta);
  for (int j = 0; j < dim; ++j) p = __dmul_rn(p, delta);
  return p;
}

__device__ __forceinline__ double ball_volume(int dim, double r) {
  const double pi = 3.141592653589793238462643383279502884;
  if (dim == 1) return __dmul_rn(2.0, r);
  if (dim == 2) return __dmul_rn(__dmul_rn(pi, r), r);
  return __dmul_rn(__dmul_rn(__dmul_rn(4.0 / 3.0 * pi, r), r), r);
}

// MatchedPolynomial::operator() — Horner in s^2 (kernel.cpp:106-112).
__device__ __forceinline__ double poly_eval(const Profile& p, double s) {
  const double t = __dmul_rn(s, s);
  double acc = 0.0;
  for (int j = p.npoly - 1; j >= 0; --j) acc = __dadd_rn(__dmul_rn(acc, t), p.poly[j]);
  return acc;
}

// SplitKernel::kappa (kernel.cpp:114-126), including the factored edge branch.
__device__ __forceinline__ double kappa_eval(const Profile& p, double s) {
  s = fabs(s);
  if (s >= 1.0) return 0.0;
  if (s < 0.5) return __dsub_rn(__ddiv_rn(p.c, s), poly_eval(p, s));
  const double u = __dsub_rn(1.0, s);
  double f = 1.0;
  for (int i = 0; i <= p.order; ++i) f = __dmul_rn(f, u);
  double acc = 0.0;
  for (int j = p.ntail - 1; j >= 0; --j) acc = __dadd_rn(__dmul_rn(acc, s), p.tail[j]);
  return __ddiv_rn(__dmul_rn(f, acc), s);
}

// eval_profile (kernel.cpp:164-182); families as in include/nlgpu.h.
__device__ __forceinline__ double profile_eval(const Profile& p, double s) {
  s = fabs(s);
  if (s >= 1.0) return 0.0;
  switch (p.family) {
    case 1: return __ddiv_rn(p.c, s);                                   // InverseS
    case 2: return __dmul_rn(__ddiv_rn(p.c, s), __dsub_rn(1.0, s));     // Conical
    case 3: return kappa_eval(p, s);                                    // Regularized
    case 0: return poly_eval(p, s);                                     // Truncated
    default: return 0.0;
  }
}

// Double-double helpers for compensated prefix sums.
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const double lo = __dadd_rn(__dadd_rn(s.lo, a.lo), b.lo);
  return two_sum(s.hi, lo);
}
__device__ __forceinline__ dd dd_sub(dd a, dd b) { return dd_add(a, {-b.hi, -b.lo}); }
__device__ __forceinline__ double dd_val(dd a) { return __dadd_rn(a.hi, a.lo); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace nlg
