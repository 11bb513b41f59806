// paper_1905_08375_b200/csrc/direct.cu — direct-sum applies (the in-repo
// GPU oracle and the compute-bound fp64 kernel).
//
// One thread per target node; the thread walks the window around its node
// (a superset of window_around, operators.cpp:31-42) and applies the exact
// inclusion predicate of the route it reproduces:
//   KIND 0  apply_truncated_dense  operators.cpp:169-204 (Leaf/Point, Mass/Difference, self included)
//   KIND 1  apply_smooth_dense     operators.cpp:206-234 (Point, self skipped, kappa profile)
//   KIND 2  apply_full_dense       operators.cpp:236-260 with eval_omega kernel.cpp:275-287
//   KIND 3  BASELINE fractional    omega = C(x) kw(x,y) |y-x|^-alpha, Point rule
//   KIND 4  BASELINE peridynamics  -h^d sum C(x)/|r| (e.(u_y-u_x)) e, Point rule
// Exterior: clip (reference) or zero collar (u = 0 outside, kappa_y := kappa_x,
// delta_y := delta_x outside).
#include <cmath>
#include <vector>

#include "plan.hpp"

namespace nlg {

namespace {

struct DirectArgs {
  Geom g;
  Profile p;
  const double* u;
  const double* delta;
  double delta0;
  const double* coeff;
  double coeff0;
  const double* kappa;
  double reach;
  int rule, form, exterior, divergence;
  const int64_t* targets;
  int64_t ntargets;
  double* out;
  unsigned long long* pairs;
  const double2* wfrac;   // KIND 3 weight table: (|d h|^-alpha, 1 / (d h)^2) by |d| (1-D) or |d|^2
  int64_t wfrac_len;
};

template <int DIM>
__device__ __forceinline__ void unflatten(const Geom& g, int64_t t, int64_t* k) {
  // output-slab flat index -> global multi-index
  int64_t rest = t % g.stride0;
  k[0] = g.row_begin + t / g.stride0;
#pragma unroll
  for (int j = DIM - 1; j >= 1; --j) {
    k[j] = rest % g.n;
    rest /= g.n;
  }
}

template <int DIM>
__device__ __forceinline__ int64_t in_index(const Geom& g, const int64_t* k) {
  int64_t rest = 0;
#pragma unroll
  for (int j = 1; j < DIM; ++j) rest = rest * g.n + k[j];
  return (k[0] - g.in_begin) * g.stride0 + rest;
}

template <int DIM, int KIND>
__global__ void __launch_bounds__(256) direct_kernel(DirectArgs a) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long my_pairs = 0;
  if (t < a.ntargets) {
    const Geom& g = a.g;
    const int64_t tt = a.targets ? a.targets[t] : t;
    int64_t ki[3] = {0, 0, 0};
    unflatten<DIM>(g, tt, ki);
    const int64_t ii = in_index<DIM>(g, ki);
    const double h = g.h;
    double x[3];
#pragma unroll
    for (int j = 0; j < DIM; ++j) x[j] = coord(ki[j], h);
    const double delta = a.delta ? a.delta[ii] : a.delta0;
    const double ci = a.coeff ? a.coeff[ii] : a.coeff0;
    const double kap_i = a.kappa ? a.kappa[ii] : 1.0;
    const bool collar = a.exterior == 1 && (KIND >= 2);
    const double radius = (KIND == 2 && a.reach > 0.0) ? a.reach : delta;
    const int64_t W = static_cast<int64_t>(floor(radius / h)) + 2;
    int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
#pragma unroll
    for (int j = 0; j < DIM; ++j) {
      lo[j] = ki[j] - W;
      hi[j] = ki[j] + W;
      if (!collar) {
        lo[j] = lo[j] < 0 ? 0 : lo[j];
        hi[j] = hi[j] > g.n - 1 ? g.n - 1 : hi[j];
      }
    }
    constexpr int NC = KIND == 4 ? DIM : 1;
    double ui[NC];
    const int64_t nin = (g.in_end - g.in_begin) * g.stride0;
#pragma unroll
    for (int c = 0; c < NC; ++c) ui[c] = a.u[c * nin + ii];
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    const double r2max = __dmul_rn(delta, delta);

    int64_t k[3] = {0, 0, 0};
    for (k[0] = lo[0]; k[0] <= hi[0]; ++k[0]) {
      for (k[1] = (DIM > 1 ? lo[1] : 0); k[1] <= (DIM > 1 ? hi[1] : 0); ++k[1]) {
        for (k[2] = (DIM > 2 ? lo[2] : 0); k[2] <= (DIM > 2 ? hi[2] : 0); ++k[2]) {
          bool in_dom = true;
#pragma unroll
          for (int j = 0; j < DIM; ++j) in_dom = in_dom && k[j] >= 0 && k[j] < g.n;
          bool self = true;
#pragma unroll
          for (int j = 0; j < DIM; ++j) self = self && k[j] == ki[j];
          double y[3];
#pragma unroll
          for (int j = 0; j < DIM; ++j) y[j] = coord(k[j], h);
          // dist (operators.cpp:71-78), exact op order
          double r2 = 0.0;
#pragma unroll
          for (int j = 0; j < DIM; ++j) {
            const double d = __dsub_rn(y[j], x[j]);
            r2 = __dadd_rn(r2, __dmul_rn(d, d));
          }
          const double r = __dsqrt_rn(r2);
          const int64_t kk = in_dom ? in_index<DIM>(g, k) : -1;
          if (KIND == 0) {
            bool in;
            if (a.rule == 1) {
              in = r < delta;
            } else {
              // cube_intersects_ball on the leaf box (geometry.cpp:63-76)
              double dmin = 0.0;
#pragma unroll
              for (int j = 0; j < DIM; ++j) {
                const double blo = __dmul_rn(static_cast<double>(k[j]), h);
                const double bhi = __dmul_rn(static_cast<double>(k[j] + 1), h);
                if (blo > x[j]) {
                  const double d = __dsub_rn(blo, x[j]);
                  dmin = __dadd_rn(dmin, __dmul_rn(d, d));
                } else if (bhi < x[j]) {
                  const double d = __dsub_rn(bhi, x[j]);
                  dmin = __dadd_rn(dmin, __dmul_rn(d, d));
                }
              }
              in = dmin < r2max;
            }
            if (!in) continue;
            ++my_pairs;
            const double v = poly_eval(a.p, __ddiv_rn(r, delta));
            acc[0] += a.form == 0 ? v * a.u[kk] : v * (a.u[kk] - ui[0]);
          } else if (KIND == 1) {
            if (self) continue;
            if (r >= delta) continue;
            ++my_pairs;
            const double front = __ddiv_rn(1.0, delta_power(DIM, delta));
            acc[0] += ci * front * kappa_eval(a.p, __ddiv_rn(r, delta)) * (a.u[kk] - ui[0]);
          } else if (KIND == 2) {
            if (self) continue;
            double dl = delta;
            if (a.divergence) {
              const double dk = in_dom ? (a.delta ? a.delta[kk] : a.delta0) : delta;
              dl = __dmul_rn(0.5, __dadd_rn(delta, dk));
            }
            if (r >= dl) continue;
            double c = ci;
            if (a.kappa) c = c * (0.5 * (kap_i + (in_dom ? a.kappa[kk] : kap_i)));
            const double w = __dmul_rn(__ddiv_rn(c, delta_power(DIM, dl)),
                                       profile_eval(a.p, __ddiv_rn(r, dl)));
            if (w == 0.0) continue;
            ++my_pairs;
            acc[0] += w * ((in_dom ? a.u[kk] : 0.0) - ui[0]);
          } else if (KIND == 3) {
            if (self) continue;
            if (!(r < delta)) continue;
            ++my_pairs;
            double c = ci;
            if (a.kappa) c = c * (0.5 * (kap_i + (in_dom ? a.kappa[kk] : kap_i)));
            const double w = c * pow(r, -a.p.alpha);
            acc[0] += w * ((in_dom ? a.u[kk] : 0.0) - ui[0]);
          } else {
            if (self) continue;
            if (!(r < delta)) continue;
            ++my_pairs;
            double e[3];
            double proj = 0.0;
#pragma unroll
            for (int j = 0; j < NC; ++j) {
              e[j] = __ddiv_rn(__dsub_rn(y[j], x[j]), r);
              const double du = (in_dom ? a.u[j * nin + kk] : 0.0) - ui[j];
              proj += e[j] * du;
            }
            const double w = __ddiv_rn(ci, r);
#pragma unroll
            for (int j = 0; j < NC; ++j) acc[j] += w * proj * e[j];
          }
        }
      }
    }
    const int64_t nout = a.targets ? a.ntargets : (g.row_end - g.row_begin) * g.stride0;
    if (KIND == 0) {
      const double front = __ddiv_rn(ci, delta_power(DIM, delta));
      a.out[t] = a.form == 0 ? front * (g.hd * acc[0] - ball_volume(DIM, delta) * ui[0])
                             : front * g.hd * acc[0];
    } else if (KIND == 4) {
#pragma unroll
      for (int c = 0; c < NC; ++c) a.out[c * nout + t] = -g.hd * acc[c];
    } else {
      a.out[t] = g.hd * acc[0];
    }
  }
  if (a.pairs) {
    my_pairs = warp_sum(my_pairs);
    if ((threadIdx.x & 31) == 0 && my_pairs) atomicAdd(a.pairs, my_pairs);
  }
}

// KIND 3 (the BASELINE fractional operator) with the per-pair work cut to
// the algorithmic minimum. Same inclusion set and pair count as direct_kernel:
// integer |d|^2 decides every candidate outside the tie band (m_lo, m_hi
// around (delta/h)^2, common.cuh tie_band), the reference's float predicate
// sqrt(r2) < delta (operators.cpp:71-78) the ones inside it; each row of the
// window is cut to |d_last|^2 <= m_hi - (the other components), so no
// candidate outside the ball is visited. The weight |r|^-alpha comes from a
// plan table at the exact lattice distance, w(m) = |d h|^-alpha, corrected to
// the float r2 of the node coordinates to first order,
//   |r|^-alpha = w(m) (1 - alpha/2 (r2 / r2(m) - 1)),
// (exact when the coordinates are exact, e.g. n = 2^L; the neglected term is
// ~ (alpha r2 rel err)^2 ~ 1e-26 otherwise) instead of a pow() per pair
// (profiles/r02_direct_cfg2_ncu_full.json: 52 DFMA per pair before).
template <int DIM>
__global__ void __launch_bounds__(256) direct_frac_kernel(const __grid_constant__ DirectArgs a) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long my_pairs = 0;
  if (t < a.ntargets) {
    const Geom& g = a.g;
    const int64_t tt = a.targets ? a.targets[t] : t;
    int64_t ki[3] = {0, 0, 0};
    unflatten<DIM>(g, tt, ki);
    const int64_t ii = in_index<DIM>(g, ki);
    const double h = g.h, inv_h = 1.0 / h;
    double x[3];
#pragma unroll
    for (int j = 0; j < DIM; ++j) x[j] = coord(ki[j], h);
    const double delta = a.delta ? a.delta[ii] : a.delta0;
    const double ci = a.coeff ? a.coeff[ii] : a.coeff0;
    const double kap_i = a.kappa ? a.kappa[ii] : 1.0;
    const bool collar = a.exterior == 1;
    const double e = delta * inv_h, e2 = e * e;
    const int64_t mlo = static_cast<int64_t>(ceil(e2 * (1.0 - tie_band_n(inv_h))));
    const int64_t mhi = static_cast<int64_t>(floor(e2 * (1.0 + tie_band_n(inv_h))));
    const double ui = a.u[ii];
    const double ca = 0.5 * a.p.alpha;
    // sum w (u_y - u_i), w = ci (kappa_i + kappa_y)/2 |r|^-alpha:  A = sum w0 (u_y - u_i),
    // B = sum w0 kappa_y (u_y - u_i)  (w0 = |r|^-alpha), out = h^d ci (kappa_i A + B) / 2
    double A = 0.0, Bk = 0.0;
    // one row of the window along the last axis: k_last in [c0, c1], the other
    // components fixed (their squared float distance r2o summed first, in the
    // reference's dimension order, and their squared lattice distance mo)
    // the reference's predicate sqrt_rn(r2) < delta as r2 < thr (sqrt_rn is
    // monotone; thr = the smallest double whose rounded root reaches delta)
    double thr = __dmul_rn(delta, delta);
    while (thr > 0.0 && __dsqrt_rn(thr) >= delta) thr = __longlong_as_double(__double_as_longlong(thr) - 1);
    while (__dsqrt_rn(thr) < delta) thr = __longlong_as_double(__double_as_longlong(thr) + 1);
    const double xl = x[DIM - 1];
    const int kil = static_cast<int>(ki[DIM - 1]);
    const int nl = static_cast<int>(g.n);
    const int mlo32 = static_cast<int>(mlo);
    // one row of the window along the last axis: k_last in [c0, c1], the other
    // components fixed (their squared float distance r2o summed first, in the
    // reference's dimension order, and their squared lattice distance mo)
    auto row = [&](const int64_t* ko, double r2o, int64_t mo, bool dom_o, int64_t c0, int64_t c1) {
      constexpr int L = DIM - 1;
      int64_t base = 0;   // input index of k_last = 0 on this row
      if (DIM > 1) {
        int64_t rest = 0;
#pragma unroll
        for (int j = 1; j < L; ++j) rest = rest * g.n + ko[j];
        base = DIM == 2 ? (ko[0] - g.in_begin) * g.stride0 : (ko[0] - g.in_begin) * g.stride0 + rest * g.n;
      } else {
        base = -g.in_begin;
      }
      const double* __restrict__ ur = a.u + base;
      const double* __restrict__ kr = a.kappa ? a.kappa + base : nullptr;
      const int mo32 = static_cast<int>(mo);
      for (int kl = static_cast<int>(c0); kl <= static_cast<int>(c1); ++kl) {
        const int dl = kl - kil, m = mo32 + dl * dl;
        if (m == 0) continue;
        const double d = __dsub_rn(__dmul_rn(__dadd_rn(static_cast<double>(kl), 0.5), h), xl);
        const double r2 = __dadd_rn(r2o, __dmul_rn(d, d));
        if (m >= mlo32 && !(r2 < thr)) continue;                    // tie band: the reference's predicate
        const double2 wt = __ldg(a.wfrac + (DIM == 1 ? (dl < 0 ? -dl : dl) : m));
        const double w0 = fma(-ca * fma(r2, wt.y, -1.0), wt.x, wt.x);
        ++my_pairs;
        const bool in_dom = dom_o && kl >= 0 && kl < nl;
        const double du = (in_dom ? ur[kl] : 0.0) - ui;              // difference form, as the reference
        A = fma(w0, du, A);
        if (kr) Bk = fma(w0 * (in_dom ? kr[kl] : kap_i), du, Bk);
      }
    };
    auto isq = [](int64_t m) {
      int64_t r = static_cast<int64_t>(sqrt(static_cast<double>(m)));
      while (r * r > m) --r;
      while ((r + 1) * (r + 1) <= m) ++r;
      return r;
    };
    const int64_t W = isq(mhi);
    int64_t k[3] = {0, 0, 0};
    auto lo_of = [&](int j, int64_t r) { const int64_t v = ki[j] - r; return collar ? v : (v < 0 ? 0 : v); };
    auto hi_of = [&](int j, int64_t r) { const int64_t v = ki[j] + r; return collar ? v : (v > g.n - 1 ? g.n - 1 : v); };
    if (DIM == 1) {
      row(k, 0.0, 0, true, lo_of(0, W), hi_of(0, W));
    } else if (DIM == 2) {
      for (k[0] = lo_of(0, W); k[0] <= hi_of(0, W); ++k[0]) {
        const int64_t d0 = k[0] - ki[0], b = mhi - d0 * d0;
        if (b < 0) continue;
        const int64_t X = isq(b);
        const double e0 = __dsub_rn(coord(k[0], h), x[0]);
        row(k, __dmul_rn(e0, e0), d0 * d0, k[0] >= 0 && k[0] < g.n, lo_of(1, X), hi_of(1, X));
      }
    } else {
      for (k[0] = lo_of(0, W); k[0] <= hi_of(0, W); ++k[0]) {
        const int64_t d0 = k[0] - ki[0], b0 = mhi - d0 * d0;
        if (b0 < 0) continue;
        const int64_t Y = isq(b0);
        const double e0 = __dsub_rn(coord(k[0], h), x[0]);
        const double s0 = __dmul_rn(e0, e0);
        for (k[1] = lo_of(1, Y); k[1] <= hi_of(1, Y); ++k[1]) {
          const int64_t d1 = k[1] - ki[1], b1 = b0 - d1 * d1;
          if (b1 < 0) continue;
          const int64_t X = isq(b1);
          const double e1 = __dsub_rn(coord(k[1], h), x[1]);
          row(k, __dadd_rn(s0, __dmul_rn(e1, e1)), d0 * d0 + d1 * d1,
              k[0] >= 0 && k[0] < g.n && k[1] >= 0 && k[1] < g.n, lo_of(2, X), hi_of(2, X));
        }
      }
    }
    const double acc = a.kappa ? 0.5 * ci * fma(kap_i, A, Bk) : ci * A;
    a.out[t] = g.hd * acc;
  }
  if (a.pairs) {
    my_pairs = warp_sum(my_pairs);
    if ((threadIdx.x & 31) == 0 && my_pairs) atomicAdd(a.pairs, my_pairs);
  }
}

template <int DIM>
void launch_dim(int kind, const DirectArgs& a, cudaStream_t s) {
  const int threads = 256;
  const unsigned blocks = static_cast<unsigned>((a.ntargets + threads - 1) / threads);
  if (blocks == 0) return;
  switch (kind) {
    case 0: direct_kernel<DIM, 0><<<blocks, threads, 0, s>>>(a); break;
    case 1: direct_kernel<DIM, 1><<<blocks, threads, 0, s>>>(a); break;
    case 2: direct_kernel<DIM, 2><<<blocks, threads, 0, s>>>(a); break;
    case 3:
      if (a.wfrac) direct_frac_kernel<DIM><<<blocks, threads, 0, s>>>(a);
      else direct_kernel<DIM, 3><<<blocks, threads, 0, s>>>(a);
      break;
    default: direct_kernel<DIM, 4><<<blocks, threads, 0, s>>>(a); break;
  }
}

// ---- matrix view of the direct operators: transpose apply and dense assembly
// The operator is out = A u with, for KIND 1-3, A_ik = h^d w_ik (k != i, pair
// included from row i's side: row i's horizon, coefficient and rule) and
// A_ii = -h^d sum_k w_ik (exterior collar nodes included); for KIND 0 (the
// truncated operator) A_ik = h^d front_i p(r/delta_i) on the rule's set S_i
// (self included) and A_ii = h^d front_i p(0)[i in S_i] - front_i |B| (Mass) or
// -h^d sum_{k != i} A_ik / h^d (Difference). Rounding follows the products
// above, not the forward kernel's accumulation order.
template <int DIM>
struct RowInfo {
  int64_t k[3];
  double x[3];
  double delta, ci, kap;
};

template <int DIM>
__device__ __forceinline__ RowInfo<DIM> row_info(const DirectArgs& a, const int64_t* k) {
  RowInfo<DIM> R;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    R.k[j] = j < DIM ? k[j] : 0;
    R.x[j] = j < DIM ? coord(k[j], a.g.h) : 0.0;
  }
  const int64_t ii = in_index<DIM>(a.g, k);
  R.delta = a.delta ? a.delta[ii] : a.delta0;
  R.ci = a.coeff ? a.coeff[ii] : a.coeff0;
  R.kap = a.kappa ? a.kappa[ii] : 1.0;
  return R;
}

// weight w of the pair (row R, column k) without the h^d factor; false if the
// pair is not in row R's set. Self pairs: only KIND 0 (its set may hold i).
template <int DIM, int KIND>
__device__ __forceinline__ bool pair_weight(const DirectArgs& a, const RowInfo<DIM>& R, const int64_t* k, bool in_dom,
                                            int64_t kk, double& w) {
  const double h = a.g.h;
  bool self = true;
  double r2 = 0.0;
  double y[3];
#pragma unroll
  for (int j = 0; j < DIM; ++j) {
    self = self && k[j] == R.k[j];
    y[j] = coord(k[j], h);
    const double d = __dsub_rn(y[j], R.x[j]);
    r2 = __dadd_rn(r2, __dmul_rn(d, d));
  }
  const double r = __dsqrt_rn(r2);
  if (KIND == 0) {
    bool in;
    if (a.rule == 1) {
      in = r < R.delta;
    } else {
      double dmin = 0.0;
#pragma unroll
      for (int j = 0; j < DIM; ++j) {
        const double blo = __dmul_rn(static_cast<double>(k[j]), h);
        const double bhi = __dmul_rn(static_cast<double>(k[j] + 1), h);
        if (blo > R.x[j]) {
          const double d = __dsub_rn(blo, R.x[j]);
          dmin = __dadd_rn(dmin, __dmul_rn(d, d));
        } else if (bhi < R.x[j]) {
          const double d = __dsub_rn(bhi, R.x[j]);
          dmin = __dadd_rn(dmin, __dmul_rn(d, d));
        }
      }
      in = dmin < __dmul_rn(R.delta, R.delta);
    }
    if (!in) return false;
    w = __ddiv_rn(R.ci, delta_power(DIM, R.delta)) * poly_eval(a.p, __ddiv_rn(r, R.delta));
    return true;
  }
  if (self) return false;
  if (KIND == 1) {
    if (r >= R.delta) return false;
    w = R.ci * __ddiv_rn(1.0, delta_power(DIM, R.delta)) * kappa_eval(a.p, __ddiv_rn(r, R.delta));
    return true;
  }
  if (KIND == 2) {
    double dl = R.delta;
    if (a.divergence) {
      const double dk = in_dom ? (a.delta ? a.delta[kk] : a.delta0) : R.delta;
      dl = __dmul_rn(0.5, __dadd_rn(R.delta, dk));
    }
    if (r >= dl) return false;
    double c = R.ci;
    if (a.kappa) c = c * (0.5 * (R.kap + (in_dom ? a.kappa[kk] : R.kap)));
    w = __dmul_rn(__ddiv_rn(c, delta_power(DIM, dl)), profile_eval(a.p, __ddiv_rn(r, dl)));
    return w != 0.0;
  }
  // KIND 3 (BASELINE fractional)
  if (!(r < R.delta)) return false;
  double c = R.ci;
  if (a.kappa) c = c * (0.5 * (R.kap + (in_dom ? a.kappa[kk] : R.kap)));
  w = c * pow(r, -a.p.alpha);
  return true;
}

// window half-width (cells) of row R
template <int DIM, int KIND>
__device__ __forceinline__ int64_t row_window(const DirectArgs& a, double delta) {
  const double radius = (KIND == 2 && a.reach > 0.0) ? a.reach : delta;
  return static_cast<int64_t>(floor(radius / a.g.h)) + 2;
}

// diagonal entry A_ii (with h^d) by enumerating row i
template <int DIM, int KIND>
__device__ double row_diag(const DirectArgs& a, const RowInfo<DIM>& R) {
  const Geom& g = a.g;
  const bool collar = a.exterior == 1 && KIND >= 2;
  const int64_t W = row_window<DIM, KIND>(a, R.delta);
  int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
#pragma unroll
  for (int j = 0; j < DIM; ++j) {
    lo[j] = R.k[j] - W;
    hi[j] = R.k[j] + W;
    if (!collar) {
      lo[j] = lo[j] < 0 ? 0 : lo[j];
      hi[j] = hi[j] > g.n - 1 ? g.n - 1 : hi[j];
    }
  }
  double sum = 0.0, self = 0.0;
  int64_t k[3] = {0, 0, 0};
  for (k[0] = lo[0]; k[0] <= hi[0]; ++k[0])
    for (k[1] = (DIM > 1 ? lo[1] : 0); k[1] <= (DIM > 1 ? hi[1] : 0); ++k[1])
      for (k[2] = (DIM > 2 ? lo[2] : 0); k[2] <= (DIM > 2 ? hi[2] : 0); ++k[2]) {
        bool in_dom = true, isself = true;
#pragma unroll
        for (int j = 0; j < DIM; ++j) {
          in_dom = in_dom && k[j] >= 0 && k[j] < g.n;
          isself = isself && k[j] == R.k[j];
        }
        const int64_t kk = in_dom ? in_index<DIM>(g, k) : -1;
        double w;
        if (!pair_weight<DIM, KIND>(a, R, k, in_dom, kk, w)) continue;
        if (isself) self = w;
        else sum += w;
      }
  if (KIND == 0) {
    const double front = __ddiv_rn(R.ci, delta_power(DIM, R.delta));
    return a.form == 0 ? g.hd * self - front * ball_volume(DIM, R.delta) : -g.hd * sum;
  }
  return -g.hd * sum;
}

// (A^T v)_j, one thread per output column j (this plan's output rows); rows i
// range over the input slab within the widest horizon
template <int DIM, int KIND>
__global__ void __launch_bounds__(128) transpose_kernel(DirectArgs a, double dmax) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= a.ntargets) return;
  const Geom& g = a.g;
  int64_t kj[3] = {0, 0, 0};
  unflatten<DIM>(g, t, kj);
  const int64_t jj = in_index<DIM>(g, kj);
  const RowInfo<DIM> Rj = row_info<DIM>(a, kj);
  double acc = row_diag<DIM, KIND>(a, Rj) * a.u[jj];
  const int64_t W = row_window<DIM, KIND>(a, dmax);
  int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
#pragma unroll
  for (int j = 0; j < DIM; ++j) {
    lo[j] = kj[j] - W;
    hi[j] = kj[j] + W;
    const int64_t lim_lo = j == 0 ? (g.in_begin > 0 ? g.in_begin : 0) : 0;
    const int64_t lim_hi = j == 0 ? (g.in_end < g.n ? g.in_end : g.n) - 1 : g.n - 1;
    lo[j] = lo[j] < lim_lo ? lim_lo : lo[j];
    hi[j] = hi[j] > lim_hi ? lim_hi : hi[j];
  }
  double off = 0.0;
  int64_t ki[3] = {0, 0, 0};
  for (ki[0] = lo[0]; ki[0] <= hi[0]; ++ki[0])
    for (ki[1] = (DIM > 1 ? lo[1] : 0); ki[1] <= (DIM > 1 ? hi[1] : 0); ++ki[1])
      for (ki[2] = (DIM > 2 ? lo[2] : 0); ki[2] <= (DIM > 2 ? hi[2] : 0); ++ki[2]) {
        bool isself = true;
#pragma unroll
        for (int j = 0; j < DIM; ++j) isself = isself && ki[j] == kj[j];
        if (isself) continue;
        const RowInfo<DIM> Ri = row_info<DIM>(a, ki);
        double w;
        if (!pair_weight<DIM, KIND>(a, Ri, kj, true, jj, w)) continue;
        off += w * a.u[in_index<DIM>(g, ki)];
      }
  a.out[t] = acc + g.hd * off;
}

// dense row-major matrix of an unsharded plan, one thread per row
template <int DIM, int KIND>
__global__ void __launch_bounds__(128) assemble_kernel(DirectArgs a, double* __restrict__ A, int64_t N) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const Geom& g = a.g;
  int64_t ki[3] = {0, 0, 0};
  unflatten<DIM>(g, i, ki);
  const RowInfo<DIM> R = row_info<DIM>(a, ki);
  const int64_t W = row_window<DIM, KIND>(a, R.delta);
  int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
#pragma unroll
  for (int j = 0; j < DIM; ++j) {
    lo[j] = ki[j] - W < 0 ? 0 : ki[j] - W;
    hi[j] = ki[j] + W > g.n - 1 ? g.n - 1 : ki[j] + W;
  }
  double* row = A + i * N;
  int64_t k[3] = {0, 0, 0};
  for (k[0] = lo[0]; k[0] <= hi[0]; ++k[0])
    for (k[1] = (DIM > 1 ? lo[1] : 0); k[1] <= (DIM > 1 ? hi[1] : 0); ++k[1])
      for (k[2] = (DIM > 2 ? lo[2] : 0); k[2] <= (DIM > 2 ? hi[2] : 0); ++k[2]) {
        bool isself = true;
#pragma unroll
        for (int j = 0; j < DIM; ++j) isself = isself && k[j] == ki[j];
        if (isself) continue;
        const int64_t kk = in_index<DIM>(g, k);
        double w;
        if (pair_weight<DIM, KIND>(a, R, k, true, kk, w)) row[kk] = g.hd * w;
      }
  row[i] = row_diag<DIM, KIND>(a, R);
}

template <int DIM>
void launch_matrix_dim(int kind, bool transpose, const DirectArgs& a, double dmax, double* A, int64_t N,
                       cudaStream_t s) {
  const int threads = 128;
  const int64_t work = transpose ? a.ntargets : N;
  const unsigned blocks = static_cast<unsigned>((work + threads - 1) / threads);
  if (blocks == 0) return;
#define NLG_MAT_CASE(KD)                                                           \
  case KD:                                                                         \
    if (transpose) transpose_kernel<DIM, KD><<<blocks, threads, 0, s>>>(a, dmax);  \
    else assemble_kernel<DIM, KD><<<blocks, threads, 0, s>>>(a, A, N);             \
    break;
  switch (kind) {
    NLG_MAT_CASE(0)
    NLG_MAT_CASE(1)
    NLG_MAT_CASE(2)
    NLG_MAT_CASE(3)
    default: break;
  }
#undef NLG_MAT_CASE
}

DirectArgs make_direct_args(const Plan& P, const double* u, double* out) {
  DirectArgs a;
  a.g = P.geom;
  a.p = P.prof;
  a.u = u;
  a.delta = P.d_delta;
  a.delta0 = P.delta0;
  a.coeff = P.d_coeff;
  a.coeff0 = P.coeff0;
  a.kappa = P.d_kappa;
  a.reach = P.reach;
  a.rule = P.rule;
  a.form = P.form;
  a.exterior = P.exterior;
  a.divergence = P.divergence;
  a.targets = nullptr;
  a.ntargets = P.n_out;
  a.out = out;
  a.pairs = nullptr;
  return a;
}

}  // namespace

void launch_transpose(const Plan& P, const double* v, double* out, cudaStream_t s) {
  const DirectArgs a = make_direct_args(P, v, out);
  const int kind = direct_kind(P);
  switch (P.geom.dim) {
    case 1: launch_matrix_dim<1>(kind, true, a, P.delta_max, nullptr, 0, s); break;
    case 2: launch_matrix_dim<2>(kind, true, a, P.delta_max, nullptr, 0, s); break;
    default: launch_matrix_dim<3>(kind, true, a, P.delta_max, nullptr, 0, s); break;
  }
}

void launch_assemble(const Plan& P, double* A, int64_t N, cudaStream_t s) {
  const DirectArgs a = make_direct_args(P, nullptr, nullptr);
  const int kind = direct_kind(P);
  switch (P.geom.dim) {
    case 1: launch_matrix_dim<1>(kind, false, a, P.delta_max, A, N, s); break;
    case 2: launch_matrix_dim<2>(kind, false, a, P.delta_max, A, N, s); break;
    default: launch_matrix_dim<3>(kind, false, a, P.delta_max, A, N, s); break;
  }
}

// KIND 3 weight table (direct_frac_kernel): entry i = (|r_i|^-alpha, 1 / r_i^2)
// at the lattice distance r_i = |d| h (1-D: i = |d|) or sqrt(i) h (2-D / 3-D:
// i = |d|^2), r_i^2 in the reference's rounding of h^2 d^2. Plan-time, host.
void direct_frac_setup(Plan& P) {
  if (P.family != NLG_FRACTIONAL) return;
  const int dim = P.geom.dim;
  const double h = P.geom.h;
  const double e = P.delta_max / h, e2 = e * e * (1.0 + tie_band(h));
  const int64_t W = static_cast<int64_t>(std::floor(std::sqrt(e2))) + 2;
  const int64_t len = dim == 1 ? W + 1 : static_cast<int64_t>(e2) + 2;
  if (len > (int64_t{1} << 24)) return;   // keep the pow() kernel
  std::vector<double2> tab(static_cast<size_t>(len));
  tab[0] = make_double2(0.0, 0.0);
  for (int64_t i = 1; i < len; ++i) {
    const double d2 = dim == 1 ? static_cast<double>(i) * static_cast<double>(i) : static_cast<double>(i);
    const double r2 = d2 * (h * h);
    const long double r = std::sqrt(static_cast<long double>(d2)) * static_cast<long double>(h);
    tab[i] = make_double2(static_cast<double>(std::pow(r, -static_cast<long double>(P.prof.alpha))), 1.0 / r2);
  }
  P.d_wfrac = upload_on(tab, P.stream);
  P.wfrac_len = len;
}

int direct_kind(const Plan& P) {
  if (P.family == 5) return 4;
  if (P.family == 4) return 3;
  return P.route;  // 0 truncated, 1 smooth, 2 full
}

void launch_direct(const Plan& P, const double* u, double* out, const int64_t* targets,
                   int64_t ntargets, unsigned long long* pairs, cudaStream_t s) {
  DirectArgs a;
  a.g = P.geom;
  a.p = P.prof;
  a.u = u;
  a.delta = P.d_delta;
  a.delta0 = P.delta0;
  a.coeff = P.d_coeff;
  a.coeff0 = P.coeff0;
  a.kappa = P.d_kappa;
  a.reach = P.reach;
  a.rule = P.rule;
  a.form = P.form;
  a.exterior = P.exterior;
  a.divergence = P.divergence;
  a.targets = targets;
  a.ntargets = targets ? ntargets : P.n_out;
  a.out = out;
  a.pairs = pairs;
  a.wfrac = P.d_wfrac;
  a.wfrac_len = P.wfrac_len;
  const int kind = direct_kind(P);
  switch (P.geom.dim) {
    case 1: launch_dim<1>(kind, a, s); break;
    case 2: launch_dim<2>(kind, a, s); break;
    default: launch_dim<3>(kind, a, s); break;
  }
}

}  // namespace nlg
