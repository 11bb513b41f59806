// paper_1905_08375_b200/csrc/stencil.cu — fast method 3: 2-D / 3-D BASELINE
// operators (cfg2 fractional, cfg3 peridynamics, cfg4 fractional 3-D) as an
// offset-table stencil.
//
// At BASELINE horizons (4h..12h in 2-D, 4h..8h in 3-D) the near field IS the
// operator, so the fast path is direct quadrature with everything that does
// not depend on u hoisted out of the pair loop:
//   fractional:  out_i = s_i [ kappa_i A_i + B_i - u_i diag_i ]
//                A_i = sum_{d in N_i} w(d) u_{i+d},  B_i = sum w(d) (kappa u)_{i+d},
//                w(d) = |d|^-alpha from a table, s_i = h^{d-alpha} C_i (x 1/2 with kappa)
//   peridynamic: out_i = -h^d c_i / h [ sum_{d in N_i} M(d) u_{i+d} - Mdiag_i u_i ],
//                M(d) = d d^T / |d|^3 (tables per offset), Mdiag the plan-time sum
// N_i is the Point-rule set of the reference, sqrt(|y-x|^2) < delta_i
// (operators.cpp:71-78): integer |d|^2 decides every pair except a tie band
// around (delta/h)^2 where the float predicate on the node coordinates (the
// reference's own operation order) decides — bit-exact inclusion on any grid.
// diag / Mdiag come from this kernel in MODE 1 (same sets, same tables), so a
// constant field is annihilated exactly; the zero collar adds its exterior
// nodes there (u = 0 outside, kappa_y := kappa_x).
// One thread per target (lanes along the fastest axis: coalesced L1 loads);
// rows of the ball are visited with warp-uniform spans so weight-table reads
// are shared-memory broadcasts.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "plan.hpp"

namespace nlg {

struct StencilState {
  int dim = 2, kind = 0, H = 0;        // kind 0 fractional, 1 peridynamic
  double* wtab = nullptr;               // fractional: [(H+1)^dim] |d|^-alpha by |dx|,|dy|,|dz|
  double* mtab = nullptr;               // peridynamic: [3][(2H+1)^2] Mxx, Mxy, Myy by signed offsets
  double* diag = nullptr;               // [n_out] (fractional) or [3][n_out] (peridynamic)
  double* scale = nullptr;              // [n_out]
  double* pack = nullptr;               // [n_in] double2 (u, kappa u) for kappa-weighted fractional
  size_t tab_bytes = 0;
  int ws = 0;                           // weight row stride (2-D: padded to a multiple of 4)
  BoxFft* box = nullptr;                // constant-horizon 3-D: FFT convolution + tie band (fft3.cu)
  bool scale_const = false;             // no per-node coefficient: scale[i] == scale0
  double scale0 = 0.0;
  // column-lane apply (stencil_cy_kernel): per-node horizons, sources by TMA
  bool cy = false;
  int hs = 0;                           // largest offset component any target includes
  CUtensorMap tmu, tmk;                 // boxes of the input planes of u (re-encoded when u moves) and kappa
  CUtensorMap tmu1;                     // peridynamics: the second displacement component
  const double* tmu_base = nullptr;
};

namespace {

constexpr int kTX = 32, kTY = 4;        // 128 threads, lanes along the fastest axis

struct StArgs {
  Geom g;
  int kind, kw, collar, mode, H;
  int hs;                 // column-lane apply: box halo
  int64_t plane_out;      // stride between the component planes of out / diag (the plan's n_out, also for row ranges)
  const double* u;        // [comps][n_in]
  const double2* pk;      // (u, kappa u) when kw
  const double* delta;
  double delta0;
  const double* kappa;
  const double* tab;      // weights (device)
  int tab_len;
  int ws, wp;             // weight row stride, peridynamic plane stride (doubles)
  const double* diag;
  const double* scale;
  double* out;            // [comps][n_out]
};

__device__ __forceinline__ double node_c(int64_t k, double h) { return coord(k, h); }

// smallest double x with sqrt_rn(x) >= delta: the reference's predicate
// sqrt(r2) < delta is r2 < T exactly (sqrt_rn is monotone)
__device__ __forceinline__ double sqrt_threshold(double delta) {
  double t = __dmul_rn(delta, delta);   // positive: neighbours are +-1 in the bit pattern
  while (t > 0.0 && __dsqrt_rn(t) >= delta) t = __longlong_as_double(__double_as_longlong(t) - 1);
  while (__dsqrt_rn(t) < delta) t = __longlong_as_double(__double_as_longlong(t) + 1);
  return t;
}

// exact Point-rule membership for an offset (the tie band only)
template <int DIM>
__device__ __forceinline__ bool point_in(const int64_t* ki, const int* d, double h, double delta) {
  double r2 = 0.0;
#pragma unroll
  for (int j = 0; j < DIM; ++j) {
    const double dd = __dsub_rn(node_c(ki[j] + d[j], h), node_c(ki[j], h));
    r2 = __dadd_rn(r2, __dmul_rn(dd, dd));
  }
  return __dsqrt_rn(r2) < delta;
}

template <int DIM, int KIND, int MODE, bool KW>
__global__ void __launch_bounds__(kTX * kTY) stencil_kernel(StArgs a) {
  extern __shared__ double stab[];
  for (int i = threadIdx.y * kTX + threadIdx.x; i < a.tab_len; i += kTX * kTY) stab[i] = a.tab[i];
  __syncthreads();
  const Geom& g = a.g;
  const int64_t n = g.n;
  // target: x along threadIdx.x; remaining axes from blockIdx / threadIdx.y
  const int64_t nx = DIM == 1 ? (g.row_end - g.row_begin) : n;   // targets along the fastest axis
  const int64_t bx = (nx + kTX - 1) / kTX;
  const int64_t ix = (static_cast<int64_t>(blockIdx.x) % bx) * kTX + threadIdx.x;
  const int64_t rowsOut = DIM == 1 ? 1 : (g.row_end - g.row_begin) * (DIM == 3 ? n : 1);
  const int64_t r = (static_cast<int64_t>(blockIdx.x) / bx) * kTY + threadIdx.y;   // output row (axis0 [, axis1])
  const bool live = ix < nx && r < rowsOut;
  int64_t ki[3] = {0, 0, 0};
  if (DIM == 1) {
    ki[0] = g.row_begin + (live ? ix : 0);
  } else if (DIM == 2) {
    ki[1] = live ? ix : 0;
    ki[0] = g.row_begin + (live ? r : 0);
  } else {
    ki[2] = live ? ix : 0;
    ki[0] = g.row_begin + (live ? r / n : 0);
    ki[1] = live ? r % n : 0;
  }
  auto in_index = [&](const int64_t* k) {
    int64_t rest = 0;
    for (int j = 1; j < DIM; ++j) rest = rest * n + k[j];
    return (k[0] - g.in_begin) * g.stride0 + rest;
  };
  const int64_t ii = in_index(ki);
  const int64_t oi = live ? (ki[0] - g.row_begin) * g.stride0 + (ii - (ki[0] - g.in_begin) * g.stride0) : 0;
  const double h = g.h;
  const double delta = live ? (a.delta ? a.delta[ii] : a.delta0) : 0.0;
  const double e = delta / h;                       // horizon in cells
  // integer band: m < mlo surely in, m > mhi surely out, else float predicate
  const double e2 = e * e;
  const int mlo = live ? static_cast<int>(ceil(e2 * (1.0 - tie_band(h)))) : 0;
  const int mhi = live ? static_cast<int>(floor(e2 * (1.0 + tie_band(h)))) : -1;
  const int R = live ? static_cast<int>(floor(e)) + 1 : 0;
  int Rw = R;   // warp-uniform extent
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) Rw = max(Rw, __shfl_xor_sync(0xffffffffu, Rw, o));
  const int64_t nin_total = (g.in_end - g.in_begin) * g.stride0;
  const double ki_kappa = (KW && live) ? a.kappa[ii] : 1.0;
  const int W1 = a.H + 1;

  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;   // A, B (fractional) / out_x, out_y (peri) / diag parts
  int d[3] = {0, 0, 0};
  const int zlo = DIM == 3 ? -Rw : 0, zhi = DIM == 3 ? Rw : 0;
  for (int dz = zlo; dz <= zhi; ++dz) {
    for (int dy = (DIM == 1 ? 0 : -Rw); dy <= (DIM == 1 ? 0 : Rw); ++dy) {
      const int base2 = (DIM == 3 ? dz * dz : 0) + dy * dy;
      // this lane's half span on the row (covering the tie band), warp max
      int X = -1;
      if (live && base2 <= mhi) X = static_cast<int>(floor(sqrt(static_cast<double>(mhi - base2))));
      int Xw = X;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) Xw = max(Xw, __shfl_xor_sync(0xffffffffu, Xw, o));
      if (Xw < 0) continue;
      int64_t krow[3] = {0, 0, 0};
      if (DIM == 2) {
        krow[0] = ki[0] + dy;
      } else if (DIM == 3) {
        krow[0] = ki[0] + dz;
        krow[1] = ki[1] + dy;
      }
      const bool row_in = DIM == 1 ? true
                          : DIM == 2 ? (krow[0] >= 0 && krow[0] < n)
                                     : (krow[0] >= 0 && krow[0] < n && krow[1] >= 0 && krow[1] < n);
      const int64_t rowoff = DIM == 1 ? -g.in_begin
                             : DIM == 2 ? (krow[0] - g.in_begin) * n : ((krow[0] - g.in_begin) * n + krow[1]) * n;
      const int ay = dy < 0 ? -dy : dy, az = dz < 0 ? -dz : dz;
      for (int dx = -Xw; dx <= Xw; ++dx) {
        const int m = base2 + dx * dx;
        bool in = live && m > 0 && m <= mhi && (dx >= -X && dx <= X);
        if (in && m >= mlo) {
          if (DIM == 1) { d[0] = dx; } else if (DIM == 2) { d[0] = dy; d[1] = dx; } else { d[0] = dz; d[1] = dy; d[2] = dx; }
          in = point_in<DIM>(ki, d, h, delta);
        }
        const int64_t kx = ki[DIM - 1] + dx;
        const bool dom = row_in && kx >= 0 && kx < n;
        if (!in) continue;
        if (KIND == 0) {
          const int ax = dx < 0 ? -dx : dx;
          const int ny = DIM >= 2 ? W1 : 1;
          const double w = stab[((DIM == 3 ? az : 0) * ny + (DIM >= 2 ? ay : 0)) * a.ws + dx + a.H];
          (void)ax;
          if (MODE == 0) {
            if (!dom) continue;
            const int64_t kk = rowoff + kx;
            if (KW) {
              const double2 v = a.pk[kk];
              acc0 = fma(w, v.x, acc0);
              acc1 = fma(w, v.y, acc1);
            } else {
              acc0 = fma(w, __ldg(a.u + kk), acc0);
            }
          } else {
            if (!dom && !a.collar) continue;
            const double kk_kappa = (KW && dom) ? a.kappa[rowoff + kx] : ki_kappa;
            acc0 += KW ? w * (ki_kappa + kk_kappa) : w;
          }
        } else {
          // peridynamic 2-D: M(d) = d d^T / |d|^3, tables by signed offset
          const int t = (dy + a.H) * a.ws + (dx + a.H);
          const double mxx = stab[t], mxy = stab[a.wp + t], myy = stab[2 * a.wp + t];
          if (MODE == 0) {
            if (!dom) continue;
            const int64_t kk = rowoff + kx;
            const double ux = __ldg(a.u + kk), uy = __ldg(a.u + nin_total + kk);
            acc0 = fma(mxx, ux, fma(mxy, uy, acc0));
            acc1 = fma(mxy, ux, fma(myy, uy, acc1));
          } else {
            if (!dom && !a.collar) continue;
            acc0 += mxx;
            acc1 += mxy;
            acc2 += myy;
          }
        }
      }
    }
  }
  if (!live) return;
  const int64_t nout = a.plane_out;
  if (KIND == 0) {
    if (MODE == 1) {
      a.out[oi] = acc0;
    } else {
      const double ui = KW ? a.pk[ii].x : a.u[ii];
      const double X = KW ? fma(ki_kappa, acc0, acc1) : acc0;
      a.out[oi] = a.scale[oi] * (X - ui * a.diag[oi]);
    }
  } else {
    if (MODE == 1) {
      a.out[oi] = acc0;
      a.out[nout + oi] = acc1;
      a.out[2 * nout + oi] = acc2;
    } else {
      const double ux = a.u[ii], uy = a.u[nin_total + ii];
      const double dxx = a.diag[oi], dxy = a.diag[nout + oi], dyy = a.diag[2 * nout + oi];
      const double s = a.scale[oi];
      a.out[oi] = s * (acc0 - (dxx * ux + dxy * uy));
      a.out[nout + oi] = s * (acc1 - (dxy * ux + dyy * uy));
    }
  }
}

// ---- apply (MODE 0) ---------------------------------------------------------
// One thread per target; the thread walks its own ball row by row with exact
// half spans (integer bound from a single-precision sqrt; only when the tie
// band around (delta/h)^2 is non-empty are the span ends re-checked with the
// reference's float predicate), and each row is ONE loop over [-xm, xp] with a
// symmetric weight row (the origin weight is 0, so the self term needs no
// branch): value load, weight load, FMA(s). 2-D: the CTA's (32+2H) x (8+2H)
// neighbourhood is staged in shared memory (zeros outside the domain: clip and
// collar apply paths coincide, the collar lives in diag). 3-D: sources via L1.

__device__ __forceinline__ int isqrt_floor(int m) {
  if (m < 0) return -1;
  int x = static_cast<int>(sqrtf(static_cast<float>(m)));
  if (x * x > m) --x;
  else if ((x + 1) * (x + 1) <= m) ++x;
  return x;
}

template <int DIM>
struct Ball {
  int mlo, mhi;
  bool tie;          // non-empty tie band [mlo, mhi]
  int64_t ki[3];
  double h, delta;
  __device__ __forceinline__ void init(double dl, double hh) {
    delta = dl;
    h = hh;
    const double e = dl / hh, e2 = e * e;
    mlo = static_cast<int>(ceil(e2 * (1.0 - tie_band(hh))));
    mhi = static_cast<int>(floor(e2 * (1.0 + tie_band(hh))));
    tie = mlo <= mhi;
  }
  __device__ __forceinline__ bool in(const int* d) const {
    int m = 0;
#pragma unroll
    for (int j = 0; j < DIM; ++j) m += d[j] * d[j];
    if (m == 0 || m > mhi) return false;
    if (m < mlo) return true;
    return point_in<DIM>(ki, d, h, delta);
  }
  // exact half spans of the row with leading offsets d[0..DIM-2]; false if empty
  __device__ __forceinline__ bool span(int* d, int& xm, int& xp) const {
    int base2 = 0;
#pragma unroll
    for (int j = 0; j < DIM - 1; ++j) base2 += d[j] * d[j];
    const int X = isqrt_floor(mhi - base2);
    if (X < 0) return false;
    xp = X;
    xm = X;
    if (tie && base2 + X * X >= mlo) {
      d[DIM - 1] = xp;
      while (xp > 0 && !in(d)) { --xp; d[DIM - 1] = xp; }
      d[DIM - 1] = -xm;
      while (xm > 0 && !in(d)) { --xm; d[DIM - 1] = -xm; }
      if (base2 != 0) {
        d[DIM - 1] = 0;
        if (!in(d)) return false;
      }
    }
    return true;
  }
};

template <bool KW>
__device__ __forceinline__ void row_sum(const double2* v, const double* w, int xm, int xp, double& a0, double& a1) {
  double s0 = 0.0, s1 = 0.0, t0 = 0.0, t1 = 0.0;
  int k = -xm;
#pragma unroll 2
  for (; k + 1 <= xp; k += 2) {
    const double2 va = v[k], vb = v[k + 1];
    const double wa = w[k], wb = w[k + 1];
    s0 = fma(wa, va.x, s0);
    t0 = fma(wb, vb.x, t0);
    if (KW) {
      s1 = fma(wa, va.y, s1);
      t1 = fma(wb, vb.y, t1);
    }
  }
  if (k <= xp) {
    const double2 va = v[k];
    s0 = fma(w[k], va.x, s0);
    if (KW) s1 = fma(w[k], va.y, s1);
  }
  a0 += s0 + t0;
  if (KW) a1 += s1 + t1;
}

// 2-D apply, register-blocked. A warp owns a patch of kLY target rows x
// kLX * kRX columns; each lane kRX adjacent targets of one row. For every ball
// row the warp sweeps the warp-uniform offset range [-XW, XW] (XW the widest
// half span among its targets on that row); per offset k it reads ONE weight
// w(dy, k) (shared-memory broadcast) and ONE new source value — the lane's
// window of kRX sources slides by one — and issues kRX unmasked FMA pairs.
// The fractional weight is even in dy, and so is every target's span, so rows
// +dy and -dy are swept together on the pre-added sources (half the FMAs).
// The sweep starts exactly at -XW: tile columns are split by (column mod 4)
// into four planes and the start phase (-XW mod 4) is a template parameter, so
// every load offset is static; the odd row stride keeps the two rows a
// quarter warp reads on disjoint banks. Afterwards each target removes the
// offsets of the sweep outside its own span (|k| > X_r, uniform loop over the
// warp's narrowest..widest span) and adds the offsets of its tie band
// ((delta/h)^2 within tie_band, common.cuh) decided by the reference's float predicate.
// R targets per lane: a warp covers 32/R lanes x R targets = 32 columns by R
// rows, a CTA 32/R warps stacked along y = 32 x 32 targets.
constexpr int kBX = 32, kBY = 32;
#ifndef NLG_R2FRAC
#define NLG_R2FRAC 8
#endif
#ifndef NLG_R2PERI
#define NLG_R2PERI 4
#endif
#ifndef NLG_R3FRAC
#define NLG_R3FRAC 8
#endif
constexpr int kR2Frac = NLG_R2FRAC, kR2Peri = NLG_R2PERI, kR3Frac = NLG_R3FRAC;   // targets per lane

// 2-D fractional tiles may be NLG_BX2 columns wide (64: two CTAs of 8 warps per
// SM instead of three of 4, a smaller halo share); every other variant 32
#ifndef NLG_BX2
#define NLG_BX2 32
#endif
#ifndef NLG_BX3
#define NLG_BX3 32
#endif
template <int DIM, int KIND>
__host__ __device__ constexpr int tile_bx() { return KIND != 0 ? kBX : (DIM == 2 ? NLG_BX2 : (DIM == 3 ? NLG_BX3 : kBX)); }
__host__ __device__ inline int tile_bx_rt(int dim, int kind) {
  return kind != 0 ? kBX : (dim == 2 ? NLG_BX2 : (dim == 3 ? NLG_BX3 : kBX));
}
__host__ __device__ inline int tile2d_q(int H, int bx = kBX) { return bx / 4 + 2 + H / 2; }   // slots per plane
__host__ __device__ inline int tile2d_rs(int H, int bx = kBX) { return 4 * tile2d_q(H, bx) + 1; }  // row stride in slots (odd)
__host__ __device__ inline int isq_len(int H) { return (H + 1) * (H + 1) + 1; }

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool in) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(in ? 8 : 0) : "memory");
}

__device__ __forceinline__ double2 dadd2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

template <int KIND, bool KW, int R>
struct Acc2 {
  double a0[R], a1[R];
};

// One ball row (PAIR: rows +dy and -dy on pre-added sources), 2*XW+1 offsets
// from k = -XW. tp / tm: plane-0 slot of the lane's start quad in the row(s);
// window element i (i < 4) sits at slot offset o[i] = ((ph + i) & 3) Q +
// ((ph + i) >> 2), element i + 4 one slot further; wk: weight of the first
// offset (offsets advance by one double).
template <int KIND, bool KW, int kRX, bool PAIR>
__device__ __forceinline__ void sweep_row(Acc2<KIND, KW, kRX>& A, const double2* __restrict__ tp,
                                          const double2* __restrict__ tm, const int* o,
                                          const double* __restrict__ wk, int wplane, int nsteps) {
  auto ld = [&](int off) { return PAIR ? dadd2(tp[off], tm[off]) : tp[off]; };
  double2 W[kRX + 4];
#pragma unroll
  for (int i = 0; i < kRX; ++i) W[i] = ld(o[i & 3] + (i >> 2));
  auto chunk = [&](auto mask_tag, int left) {
    constexpr bool MASK = decltype(mask_tag)::value;
#pragma unroll
    for (int j = 0; j < 4; ++j) W[kRX + j] = ld(o[j] + kRX / 4);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const bool on = !MASK || s < left;
      if (KIND == 0) {
        double w = wk[s];
        if (MASK) w = on ? w : 0.0;
#pragma unroll
        for (int r = 0; r < kRX; ++r) {
          A.a0[r] = fma(w, W[s + r].x, A.a0[r]);
          if (KW) A.a1[r] = fma(w, W[s + r].y, A.a1[r]);
        }
      } else {
        double mxx = wk[s], mxy = wk[wplane + s], myy = wk[2 * wplane + s];
        if (MASK) {
          mxx = on ? mxx : 0.0;
          mxy = on ? mxy : 0.0;
          myy = on ? myy : 0.0;
        }
#pragma unroll
        for (int r = 0; r < kRX; ++r) {
          const double2 v = W[s + r];
          A.a0[r] = fma(mxx, v.x, fma(mxy, v.y, A.a0[r]));
          A.a1[r] = fma(mxy, v.x, fma(myy, v.y, A.a1[r]));
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kRX; ++i) W[i] = W[i + 4];
    tp += 1;
    if (PAIR) tm += 1;
    wk += 4;
  };
  int left = nsteps;
  for (; left >= 8; left -= 8) {          // two chunks per trip: the window shift is register renaming
    chunk(std::false_type{}, 4);
    chunk(std::false_type{}, 4);
  }
  if (left >= 4) {
    chunk(std::false_type{}, 4);
    left -= 4;
  }
  if (left > 0) chunk(std::true_type{}, left);
}

// DIM 2: one tile of kBY x kBX targets. DIM 3: the same tile in one target
// plane z, the source planes z + dz visited one at a time (staged in shared
// memory, the in-plane sweep as in 2-D with |d|^2 budgets reduced by dz^2);
// the grid runs z fastest so the blocks in flight share their source planes
// in L2.
template <int DIM, int KIND, bool KW, int kRX>
__global__ void __launch_bounds__(tile_bx<DIM, KIND>() * kBY / kRX, (kRX == 8 ? 4 : 3) * kBX / tile_bx<DIM, KIND>())
    stencil_rb_kernel(StArgs a) {
  constexpr int kBXt = tile_bx<DIM, KIND>();
  constexpr int kLX = kBXt / kRX, kLY = 32 / kLX, kWY = kBY / kLY;
  extern __shared__ __align__(16) double sm[];
  const int H = a.H, Q = tile2d_q(H, kBXt), RS = tile2d_rs(H, kBXt), TH = kBY + 2 * H, TWc = 4 * Q;
  double2* tile = reinterpret_cast<double2*>(sm);          // [TH][RS slots: 4 planes x Q, +1 pad]
  double* wt = sm + 2 * static_cast<size_t>(TH + 1) * RS;  // row TH: zeros (partner of row 0)
  // weights in shared memory: the whole table (2-D) or the rows of the current |dz| (3-D)
  const int wlen = DIM == 2 ? a.tab_len : (H + 1) * a.ws;
  int* isq = reinterpret_cast<int*>(wt + wlen);            // isqrt table for 0..(H+1)^2
  int* bmax = isq + isq_len(H);                            // block max of M (3-D plane range)
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int i = tid; i < RS; i += 32 * kWY) tile[static_cast<size_t>(TH) * RS + i] = make_double2(0.0, 0.0);
  if (DIM == 2)
    for (int i = tid; i < wlen; i += 32 * kWY) wt[i] = a.tab[i];
  for (int i = tid; i < isq_len(H); i += 32 * kWY) {
    int x = static_cast<int>(sqrtf(static_cast<float>(i)));
    while (x * x > i) --x;
    while ((x + 1) * (x + 1) <= i) ++x;
    isq[i] = x;
  }
  if (tid == 0) *bmax = -1;
  const Geom& g = a.g;
  const int64_t n = g.n;
  // tile origin: 2-D (x0, y0) from the grid; 3-D z fastest, then the x-y tile
  int64_t x0, y0, z = 0;
  if (DIM == 2) {
    x0 = static_cast<int64_t>(blockIdx.x) * kBXt;
    y0 = g.row_begin + static_cast<int64_t>(blockIdx.y) * kBY;
  } else {
    const int64_t ntx = (n + kBXt - 1) / kBXt;
    z = g.row_begin + blockIdx.x;
    x0 = (blockIdx.y % ntx) * kBXt;
    y0 = (blockIdx.y / ntx) * kBY;   // grid.y = ntx * ceil(n / kBY)
  }
  const int64_t ystop = DIM == 2 ? g.row_end : n;
  const int64_t nin_total = (g.in_end - g.in_begin) * g.stride0;
  const int tx = threadIdx.x & (kLX - 1);                   // lane column
  const int wy = threadIdx.y * kLY + threadIdx.x / kLX;     // target row within the CTA
  const int64_t iy = y0 + wy;
  const bool yok = iy < ystop;
  const double inv_h = 1.0 / g.h;
  auto in_index = [&](int64_t ix) {
    return DIM == 2 ? (iy - g.in_begin) * n + ix : ((z - g.in_begin) * n + iy) * n + ix;
  };
  // 3-D: the epilogue's per-target operands (u, kappa, scale, diag) are
  // independent of the sweep: prefetched into L2 now, they are hits when the
  // sums are done (cfg4-B 137 -> 135 ms; in 2-D it costs more than it saves)
  if (DIM == 3 && yok && x0 + kRX * tx < n) {
    const int64_t i0 = in_index(x0 + kRX * tx), o0 = i0 - (g.row_begin - g.in_begin) * g.stride0;
    const int64_t last = min(static_cast<int64_t>(kRX - 1), n - 1 - (x0 + kRX * tx));
    const int64_t pout = a.plane_out;
    auto pf = [](const double* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); };
    for (int64_t e : {int64_t(0), last}) {
      pf(a.u + i0 + e);
      pf(a.scale + o0 + e);
      pf(a.diag + o0 + e);
      if (KW) pf(a.kappa + i0 + e);
      if (KIND == 1) {
        pf(a.u + nin_total + i0 + e);
        pf(a.diag + pout + o0 + e);
        pf(a.diag + 2 * pout + o0 + e);
      }
    }
  }
  // targets of this lane: M = largest |d|^2 surely inside (below the tie band)
  int M[kRX];
  unsigned tiem = 0;
  int Mx = -1, Mn = 1 << 20;
#pragma unroll
  for (int r = 0; r < kRX; ++r) {
    const int64_t ix = x0 + kRX * tx + r;
    M[r] = -1;
    if (yok && ix < n) {
      const int64_t ii = in_index(ix);
      const double e = (a.delta ? a.delta[ii] : a.delta0) * inv_h, e2 = e * e;
      const int mlo = static_cast<int>(ceil(e2 * (1.0 - tie_band_n(inv_h))));
      const int mhi = static_cast<int>(floor(e2 * (1.0 + tie_band_n(inv_h))));
      M[r] = mlo <= mhi ? mlo - 1 : mhi;
      if (mlo <= mhi) tiem |= 1u << r;
      Mn = min(Mn, M[r]);
    }
    Mx = max(Mx, M[r]);
  }
  const int MW = __reduce_max_sync(0xffffffffu, Mx);
  const int MN = __reduce_min_sync(0xffffffffu, Mn);
  const bool tie_const = a.delta == nullptr;
  int m0c = -1;
  double Tc = 0.0;
  if (tie_const) {
    const double e = a.delta0 * inv_h, e2 = e * e;
    const int mlo = static_cast<int>(ceil(e2 * (1.0 - tie_band_n(inv_h))));
    const int mhi = static_cast<int>(floor(e2 * (1.0 + tie_band_n(inv_h))));
    if (mlo <= mhi) {
      m0c = mlo;
      Tc = sqrt_threshold(a.delta0);
    }
  }
  __syncthreads();
  if (DIM == 3) {
    int Mt = Mx;                                 // tie bands sit at M + 1
#pragma unroll
    for (int r = 0; r < kRX; ++r)
      if (tiem >> r & 1u) Mt = max(Mt, M[r] + 1);
    Mt = __reduce_max_sync(0xffffffffu, Mt);
    if ((threadIdx.x & 31) == 0) atomicMax(bmax, Mt);
  }
  __syncthreads();
  auto isqrt_t = [&](int m) { return m < 0 ? -1 : isq[m]; };
  const int Rz = DIM == 3 ? isqrt_t(*bmax) : 0;
  Acc2<KIND, KW, kRX> A;
#pragma unroll
  for (int r = 0; r < kRX; ++r) A.a0[r] = A.a1[r] = 0.0;
  const int cy = wy + H;
  auto tv = [&](int dy, int r, int k) {
    const int c = kRX * tx + r + H + k;
    return tile[static_cast<size_t>(cy + dy) * RS + (c & 3) * Q + (c >> 2)];
  };
  auto wrow_of = [&](int az, int dy) {
    (void)az;
    const int ay = dy < 0 ? -dy : dy;
    return (KIND == 0 ? ay : dy + H) * a.ws;
  };
  auto add = [&](int r, int az, int dy, int k, double sg) {
    const double2 v = tv(dy, r, k);
    const int t = wrow_of(az, dy) + k + H;
    if (KIND == 0) {
      const double w = sg * wt[t];
      A.a0[r] = fma(w, v.x, A.a0[r]);
      if (KW) A.a1[r] = fma(w, v.y, A.a1[r]);
    } else {
      const double mxx = sg * wt[t], mxy = sg * wt[a.wp + t], myy = sg * wt[2 * a.wp + t];
      A.a0[r] = fma(mxx, v.x, fma(mxy, v.y, A.a0[r]));
      A.a1[r] = fma(mxy, v.x, fma(myy, v.y, A.a1[r]));
    }
  };
  // one plane's value at (gz, iy + dy, x_r + sx) straight from global memory
  // (3-D tie points decided differently on the two mirrored planes)
  auto lone_side = [&](int r, int dy, int sx, int64_t gz) {
    const int64_t gy = iy + dy, gx = x0 + kRX * tx + r + sx;
    if (gz < 0 || gz >= n || gz < g.in_begin || gz >= g.in_end || gy < 0 || gy >= n || gx < 0 || gx >= n) return;
    const int64_t k = ((gz - g.in_begin) * n + gy) * n + gx;
    const double w = wt[wrow_of(0, dy) + sx + H];
    const double uu = a.u[k];
    A.a0[r] = fma(w, uu, A.a0[r]);
    if (KW) A.a1[r] = fma(w, a.kappa[k] * uu, A.a1[r]);
  };
  // KIND 0 sweeps rows +ay / -ay together; row 0 pairs with the zero row TH
  auto sweep = [&](int az, int dy, int dm, int XW) {
    const int st = H - XW;                       // start column relative to the lane's first target - H
    const int ph = st & 3;
    int o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = ((ph + j) & 3) * Q + ((ph + j) >> 2);
    const double2* tp = tile + static_cast<size_t>(cy + dy) * RS + (kRX / 4) * tx + (st >> 2);
    const double2* tm = tile + static_cast<size_t>(dm) * RS + (kRX / 4) * tx + (st >> 2);
    const double* wk = wt + wrow_of(az, dy) + st;
    if (KIND == 0) sweep_row<KIND, KW, kRX, true>(A, tp, tm, o, wk, a.wp, 2 * XW + 1);
    else sweep_row<KIND, KW, kRX, false>(A, tp, tm, o, wk, a.wp, 2 * XW + 1);
  };
  // staging with cp.async (every load of a thread in flight at once; zero fill
  // outside the domain / slab): lane i of a 32-column group takes column
  // 4 (i & 7) + (i >> 3), so each quarter warp fills consecutive slots of one plane
  const int cl = 4 * (threadIdx.x & 7) + (threadIdx.x >> 3);
  auto stage = [&](int64_t gz, int az) {
    if (DIM == 3)   // this |dz|'s weight rows, in flight with the plane
      for (int i = tid; i < wlen; i += 32 * kWY) cp_async8(wt + i, a.tab + static_cast<size_t>(az) * wlen + i, true);
    const bool zin = DIM == 2 || (gz >= 0 && gz < n && gz >= g.in_begin && gz < g.in_end);
    for (int ty = threadIdx.y; ty < TH; ty += kWY) {
      const int64_t gy = y0 - H + ty;
      const bool yin = zin && gy >= 0 && gy < n && (DIM == 3 || (gy >= g.in_begin && gy < g.in_end));
      const int64_t rowk = DIM == 2 ? (gy - g.in_begin) * n : ((gz - g.in_begin) * n + gy) * n;
      double2* trow = tile + static_cast<size_t>(ty) * RS;
      for (int c0 = 0; c0 < TWc; c0 += 32) {
        const int c = c0 + cl;
        if (c >= TWc) continue;
        const int64_t gx = x0 - H + c;
        const bool in = yin && gx >= 0 && gx < n;
        const int64_t k = in ? rowk + gx : 0;
        double* dst = reinterpret_cast<double*>(trow + (c & 3) * Q + (c >> 2));
        if (KIND == 1) {
          cp_async8(dst, a.u + k, in);
          cp_async8(dst + 1, a.u + nin_total + k, in);
        } else if (KW) {
          cp_async8(dst, a.u + k, in);
          cp_async8(dst + 1, a.kappa + k, in);
        } else {
          cp_async8(dst, a.u + k, in);
          cp_async8(dst + 1, a.u + k, false);
        }
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    // own slots: (u, kappa) -> (u, kappa u); 3-D az > 0: plus the mirror plane
    // z - az (the fractional weight and every span are even in dz, so the two
    // planes are swept as one)
    const int64_t gzm = 2 * z - gz;
    const bool mirror = DIM == 3 && KIND == 0 && az > 0;
    const bool zmin = mirror && gzm >= 0 && gzm < n && gzm >= g.in_begin && gzm < g.in_end;
    if (KW || mirror) {
      for (int ty = threadIdx.y; ty < TH; ty += kWY) {
        const int64_t gy = y0 - H + ty;
        const bool yin = zmin && gy >= 0 && gy < n;
        const int64_t rowm = ((gzm - g.in_begin) * n + gy) * n;
        double2* trow = tile + static_cast<size_t>(ty) * RS;
        for (int c0 = 0; c0 < TWc; c0 += 32) {
          const int c = c0 + cl;
          if (c >= TWc) continue;
          double2* dst = trow + (c & 3) * Q + (c >> 2);
          double2 v = *dst;
          if (KW) v.y = v.y * v.x;
          const int64_t gx = x0 - H + c;
          if (yin && gx >= 0 && gx < n) {
            const double um = __ldg(a.u + rowm + gx);
            v.x = v.x + um;
            if (KW) v.y = fma(__ldg(a.kappa + rowm + gx), um, v.y);
          }
          *dst = v;
        }
      }
    }
    __syncthreads();
  };
  // 3-D: planes z +- dz staged pre-added (dz = |dz| = az); 2-D: one pass
  for (int dz = 0; dz <= Rz; ++dz) {
    const int az = dz, dz2 = dz * dz;
    if (DIM == 3) __syncthreads();               // the previous plane is consumed
    stage(z + dz, az);
    const int mW = MW - dz2, mN = MN - dz2;
    const int RyW = isqrt_t(mW);
    for (int ay = 0; ay <= RyW; ++ay) {
      const int XW = isqrt_t(mW - ay * ay), XN = MN > MW ? XW : isqrt_t(mN - ay * ay);
      if (XW < 0) continue;
      if (KIND == 0) {
        sweep(az, ay, ay == 0 ? TH : cy - ay, XW);
      } else {
        sweep(az, ay, 0, XW);
        if (ay > 0) sweep(az, -ay, 0, XW);
      }
      if (XN >= XW) continue;
      // remove the sweep's offsets outside each target's own span (warp-uniform
      // offsets k = XN+1..XW, per-target selects); spans are even in dy
      int X[kRX];
#pragma unroll
      for (int r = 0; r < kRX; ++r) X[r] = isqrt_t(M[r] - dz2 - ay * ay);
      for (int k = max(XN + 1, 0); k <= XW; ++k) {
#pragma unroll
        for (int r = 0; r < kRX; ++r) {
          if (!__any_sync(0xffffffffu, X[r] < k)) continue;
          const double sg = X[r] < k ? -1.0 : 0.0;
          for (int sd = (ay == 0 ? 0 : -ay); sd <= ay; sd += (ay == 0 ? 1 : 2 * ay)) {
            add(r, az, sd, k, sg);
            if (k > 0) add(r, az, sd, -k, sg);
          }
        }
      }
    }
    // tie band of this plane: |d|^2 = m0 exactly, decided by the reference's
    // float predicate. Constant horizon: every target shares m0 and the
    // threshold, so the warp walks the lattice points of the sphere uniformly
    // and each target tests r2 < T on its own coordinates.
    if (tie_const) {
      const int rem0 = m0c - dz2;
      if (m0c >= 0 && rem0 >= 0) {
        const int Ry = isq[rem0];
        // 3-D: the tile holds planes z+dz and z-dz added; each side has its own
        // float predicate (coordinates round differently), a lone side adds its
        // own value from global memory
        const double ddp = DIM == 3 ? __dsub_rn(coord(z + dz, g.h), coord(z, g.h)) : 0.0;
        const double ddm = DIM == 3 ? __dsub_rn(coord(z - dz, g.h), coord(z, g.h)) : 0.0;
        for (int dy = -Ry; dy <= Ry; ++dy) {
          const int rem = rem0 - dy * dy, X = isq[rem];
          if (X * X != rem || (dz == 0 && dy == 0 && X == 0)) continue;
          const double ddy = __dsub_rn(coord(iy + dy, g.h), coord(iy, g.h));
          const double yy = __dmul_rn(ddy, ddy);
          const double bp = DIM == 3 ? __dadd_rn(__dmul_rn(ddp, ddp), yy) : yy;
          const double bm = DIM == 3 ? __dadd_rn(__dmul_rn(ddm, ddm), yy) : yy;
          for (int sx = -X; sx <= X; sx += (X > 0 ? 2 * X : 1)) {
#pragma unroll
            for (int r = 0; r < kRX; ++r) {
              const int64_t ix = x0 + kRX * tx + r;
              const double ddx = __dsub_rn(coord(ix + sx, g.h), coord(ix, g.h));
              const double xx = __dmul_rn(ddx, ddx);
              const bool ip = M[r] >= 0 && __dadd_rn(bp, xx) < Tc;
              const bool im = M[r] >= 0 && __dadd_rn(bm, xx) < Tc;
              if (DIM == 2 || dz == 0 || ip == im) {
                add(r, az, dy, sx, ip ? 1.0 : 0.0);
              } else {
                lone_side(r, dy, sx, ip ? z + dz : z - dz);
              }
            }
          }
        }
      }
      continue;
    }
    // variable horizon: ties are rare; a dynamic loop over the lane's tie
    // targets into scalars, then one static scatter (keeps the accumulators in
    // registers)
    unsigned tm = tiem;
    while (tm) {
      const int rr = __ffs(tm) - 1;
      tm &= tm - 1;
      const int64_t ix = x0 + kRX * tx + rr;
      const double delta = a.delta ? a.delta[in_index(ix)] : a.delta0;
      const double e = delta * inv_h, e2 = e * e;
      const int mlo = static_cast<int>(ceil(e2 * (1.0 - tie_band_n(inv_h))));
      const int mhi = static_cast<int>(floor(e2 * (1.0 + tie_band_n(inv_h))));
      const int64_t ki[3] = {DIM == 2 ? iy : z, DIM == 2 ? ix : iy, ix};
      const int Ry = isqrt_floor(mhi - dz2);
      double t0 = 0.0, t1 = 0.0;
      for (int dy = -Ry; dy <= Ry; ++dy) {
        const int X = isqrt_floor(mhi - dz2 - dy * dy);
        const int m = dz2 + dy * dy + X * X;
        if (m < mlo || m == 0) continue;
        for (int sx = -X; sx <= X; sx += (X > 0 ? 2 * X : 1)) {
          bool in, im = false;
          if (DIM == 2) {
            const int d[2] = {dy, sx};
            in = point_in<2>(ki, d, g.h, delta);
            im = in;
          } else {
            const int d[3] = {dz, dy, sx}, dm[3] = {-dz, dy, sx};
            in = point_in<3>(ki, d, g.h, delta);
            im = dz == 0 ? in : point_in<3>(ki, dm, g.h, delta);
          }
          if (!in && !im) continue;
          double2 v;
          if (in == im) {
            v = tv(dy, rr, sx);                  // both mirrored planes (or the only one)
          } else {                               // one side: its own value from global memory
            const int64_t gz = in ? z + dz : z - dz, gy = iy + dy, gx = ix + sx;
            v = make_double2(0.0, 0.0);
            if (gz >= 0 && gz < n && gz >= g.in_begin && gz < g.in_end && gy >= 0 && gy < n && gx >= 0 && gx < n) {
              const int64_t k = ((gz - g.in_begin) * n + gy) * n + gx;
              v.x = a.u[k];
              if (KW) v.y = a.kappa[k] * v.x;
            }
          }
          const int t = wrow_of(az, dy) + sx + H;
          if (KIND == 0) {
            t0 = fma(wt[t], v.x, t0);
            if (KW) t1 = fma(wt[t], v.y, t1);
          } else {
            t0 = fma(wt[t], v.x, fma(wt[a.wp + t], v.y, t0));
            t1 = fma(wt[a.wp + t], v.x, fma(wt[2 * a.wp + t], v.y, t1));
          }
        }
      }
#pragma unroll
      for (int r = 0; r < kRX; ++r) {
        if (r == rr) {
          A.a0[r] += t0;
          A.a1[r] += t1;
        }
      }
    }
  }
  if (!yok) return;
  const int64_t plane_out = a.plane_out;
#pragma unroll
  for (int r = 0; r < kRX; ++r) {
    const int64_t ix = x0 + kRX * tx + r;
    if (ix >= n) break;
    const int64_t ii = in_index(ix);
    const int64_t oi = ii - (g.row_begin - g.in_begin) * g.stride0;
    if (KIND == 0) {
      const double X = KW ? fma(a.kappa[ii], A.a0[r], A.a1[r]) : A.a0[r];
      a.out[oi] = a.scale[oi] * (X - a.u[ii] * a.diag[oi]);
    } else {
      const double ux = a.u[ii], uy = a.u[nin_total + ii];
      const double dxx = a.diag[oi], dxy = a.diag[plane_out + oi], dyy = a.diag[2 * plane_out + oi];
      const double sc = a.scale[oi];
      a.out[oi] = sc * (A.a0[r] - (dxx * ux + dxy * uy));
      a.out[plane_out + oi] = sc * (A.a1[r] - (dxy * ux + dyy * uy));
    }
  }
}


// ---- column-lane apply (fractional, per-node horizons): stencil_cy_kernel -----
// The variable-horizon 2-D / 3-D apply (cfg2, cfg4-B). Lanes run along x (the
// contiguous axis), a lane owns kCyR consecutive targets of one column, and the
// window slides along y: for a column offset dx the lane walks dy = -YW..YW,
// one new source (rows are dense, any row pitch is conflict-free) and one
// weight (broadcast) per step feeding 2 kCyR FMAs (A and B sums). The weight is
// even in dx, so columns +dx / -dx are added while loading; in 3-D the source
// planes z +- dz are added once in shared memory (the combine pass), which
// also forms kappa u. Sources arrive as dense boxes by cp.async.bulk.tensor
// (one elected thread; zero fill outside the domain / slab from the tensor
// map's bounds = the clip exterior); the mirror planes of the next |dz| are in
// flight during the sweep of the current one. Per-target horizons: the sweep
// range is the warp's widest (M_W); steps every target of the warp includes
// (|d|^2 <= M_N) run unmasked, the others predicate each FMA pair on
// |d|^2 <= M_r (integer, exact). Tie-band targets (rare with a variable
// horizon) add their band afterwards from global memory with the reference's
// float predicate.
#ifndef NLG_CY_R
#define NLG_CY_R 8
#endif
constexpr int kCyR = NLG_CY_R;          // targets per lane: 16, 12 or 8 (5, 4, 3 ring phases)
#ifndef NLG_CY_RING
#define NLG_CY_RING 1
#endif
#ifndef NLG_CY_U
#define NLG_CY_U 4                      // steps per chunk (4 or 2): the window holds kCyR + U sources
#endif
#ifndef NLG_CY_U3
#define NLG_CY_U3 2                     // 3-D scalar kernel: sweeps are ~9 steps, 2-step chunks waste fewer masked steps
#endif
constexpr int kCyU = NLG_CY_U;          // 2-D kernels
#define NLG_CY_NPH ((NLG_CY_R + NLG_CY_U) / NLG_CY_U)   // ring phases (2-D)
#ifndef NLG_CY_MINB2
#define NLG_CY_MINB2 4                  // resident CTAs per SM the register budget allows (2-D, 3-D)
#endif
#ifndef NLG_CY_MINB3
#define NLG_CY_MINB3 3
#endif
#ifndef NLG_CY_ONEVAR
#define NLG_CY_ONEVAR 0                 // 1: every chunk through the per-target select (half the code)
#endif
#ifndef NLG_CY_STEPSEL
#define NLG_CY_STEPSEL 0                // 1: plain / selected FMAs decided per step (YN carries M_N) instead of per chunk
#endif
#ifndef NLG_CY_W2
#define NLG_CY_W2 4
#endif
#ifndef NLG_CY_W3
#define NLG_CY_W3 4
#endif
#ifndef NLG_CYP_W
#define NLG_CYP_W 4                     // peridynamic variant: warps per CTA, resident CTAs
#endif
#ifndef NLG_CYP_MINB
#define NLG_CYP_MINB 4
#endif
// box row pitches with their own instantiation: the BASELINE reaches (cfg2: 11 -> 56, cfg4-B: 7 -> 48, cfg3: 8 -> 48)
constexpr int kCyBW2 = 56, kCyBW3 = 48, kCyBWp = 48;
template <int DIM>
__host__ __device__ constexpr int cy_warps() { return DIM == 2 ? NLG_CY_W2 : NLG_CY_W3; }
inline int cy_warps_rt(int dim, int kind) { return kind == 1 ? NLG_CYP_W : (dim == 2 ? cy_warps<2>() : cy_warps<3>()); }
// column halo rounded up to even: a box that starts at an odd column (a global address that is not a
// multiple of 16 bytes) faults ("illegal instruction") on the B200
__host__ __device__ inline int cy_hx(int hs) { return (hs + 1) & ~1; }
__host__ __device__ inline int cy_bw(int hs) { return 32 + 2 * cy_hx(hs); }
__host__ __device__ inline int cy_bhl(int hs, int warps) { return warps * kCyR + 2 * hs; }
__host__ __device__ inline int cy_box(int hs, int warps) {     // doubles per swept box (3 pad rows), 128-byte multiple
  return (cy_bw(hs) * (cy_bhl(hs, warps) + 3) + 15) & ~15;
}
__host__ __device__ inline int cy_mbox(int hs, int warps) {    // mirror-plane boxes (3-D): no pad rows
  return (cy_bw(hs) * cy_bhl(hs, warps) + 15) & ~15;
}

__device__ __forceinline__ void cy_mbar_wait(unsigned mb, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(mb),
      "r"(parity)
      : "memory");
}

// one column pair (+dx / -dx; dx = 0 passes the same column twice with halved
// weights): steps dy = -YW .. YW (+ up to 3 masked overshoot steps). The
// window of kCyR + 4 sources per field lives in registers as a ring: chunk
// number PH (mod 5) finds logical element i at (i + 4 PH) mod (kCyR + 4), so
// sliding by four costs no register moves.
// BWC: the row pitch of the box as a compile-time constant (the BASELINE reaches: every window load
// then carries its row offset as an immediate), 0: the run-time pitch bw_rt
template <bool KW, int PH, int BWC, int U>
__device__ __forceinline__ void cy_chunk(double (&a0)[kCyR], double (&a1)[kCyR], const int (&M)[kCyR],
                                         double (&Wu)[kCyR + U], double (&Wk)[kCyR + U], const double*& up,
                                         const double*& um, const double*& kp, const double*& km, int bw_rt,
                                         const double*& wk, int dy0, int YW, int YN, int c0) {
  constexpr int NW = kCyR + U;
  const int BW = BWC ? BWC : bw_rt;
#pragma unroll
  for (int j = 0; j < U; ++j) {
    Wu[(kCyR + j + U * PH) % NW] = up[j * BW] + um[j * BW];
    if (KW) Wk[(kCyR + j + U * PH) % NW] = kp[j * BW] + km[j * BW];
  }
#if NLG_CY_STEPSEL
  // per step: every target of the warp includes it (|d|^2 <= M_N: plain FMAs) or the weight is
  // selected to zero per target (overshoot steps of the last chunk have |d|^2 > M_W: all zero)
  (void)YW;
#pragma unroll
  for (int s = 0; s < U; ++s) {
    const double w = wk[s];
    const int c = c0 + (dy0 + s) * (dy0 + s);
    if (c <= YN) {
#pragma unroll
      for (int r = 0; r < kCyR; ++r) {
        a0[r] = fma(w, Wu[(s + r + U * PH) % NW], a0[r]);
        if (KW) a1[r] = fma(w, Wk[(s + r + U * PH) % NW], a1[r]);
      }
    } else {
#pragma unroll
      for (int r = 0; r < kCyR; ++r) {
        const double wr = c <= M[r] ? w : 0.0;
        a0[r] = fma(wr, Wu[(s + r + U * PH) % NW], a0[r]);
        if (KW) a1[r] = fma(wr, Wk[(s + r + U * PH) % NW], a1[r]);
      }
    }
  }
#else
  if (!NLG_CY_ONEVAR && dy0 >= -YN && min(dy0 + U - 1, YW) <= YN) {   // every step of the chunk inside every target's ball
#pragma unroll
    for (int s = 0; s < U; ++s) {
      const double w = dy0 + s <= YW ? wk[s] : 0.0;   // overshoot steps of the last chunk
#pragma unroll
      for (int r = 0; r < kCyR; ++r) {
        a0[r] = fma(w, Wu[(s + r + U * PH) % NW], a0[r]);
        if (KW) a1[r] = fma(w, Wk[(s + r + U * PH) % NW], a1[r]);
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < U; ++s) {
      const double w = wk[s];
      const int c = c0 + (dy0 + s) * (dy0 + s);
#pragma unroll
      for (int r = 0; r < kCyR; ++r) {   // the weight selected to zero outside the target's own ball
        const double wr = c <= M[r] ? w : 0.0;
        a0[r] = fma(wr, Wu[(s + r + U * PH) % NW], a0[r]);
        if (KW) a1[r] = fma(wr, Wk[(s + r + U * PH) % NW], a1[r]);
      }
    }
  }
#endif
  up += U * BW;
  um += U * BW;
  kp += U * BW;
  km += U * BW;
  wk += U;
}

template <bool KW, int BWC, int U>
__device__ __forceinline__ void cy_sweep(double (&a0)[kCyR], double (&a1)[kCyR], const int (&M)[kCyR],
                                         const double* up, const double* um, const double* kp, const double* km,
                                         int bw_rt, const double* wk, int YW, int YN, int c0) {
  const int BW = BWC ? BWC : bw_rt;
  double Wu[kCyR + U], Wk[kCyR + U];
#pragma unroll
  for (int i = 0; i < kCyR; ++i) {
    Wu[i] = up[i * BW] + um[i * BW];
    if (KW) Wk[i] = kp[i * BW] + km[i * BW];
  }
  up += kCyR * BW;
  um += kCyR * BW;
  kp += kCyR * BW;
  km += kCyR * BW;
  const int nsteps = 2 * YW + 1;
  int s0 = 0;
#define NLG_CY_CHUNK(PH)                                                                   \
  cy_chunk<KW, PH, BWC, U>(a0, a1, M, Wu, Wk, up, um, kp, km, BW, wk, s0 - YW, YW, YN, c0);   \
  s0 += U;                                                                              \
  if (s0 >= nsteps) break;
#if NLG_CY_RING
  for (;;) {
    NLG_CY_CHUNK(0)
    NLG_CY_CHUNK(1)
    NLG_CY_CHUNK(2)
    if constexpr ((kCyR + U) / U >= 4) {
      NLG_CY_CHUNK(3)
    }
    if constexpr ((kCyR + U) / U >= 5) {
      NLG_CY_CHUNK(4)
    }
  }
#else
  for (;;) {   // one chunk body, the window shifted by register moves
    NLG_CY_CHUNK(0)
#pragma unroll
    for (int i = 0; i < kCyR; ++i) {
      Wu[i] = Wu[i + U];
      if (KW) Wk[i] = Wk[i + U];
    }
  }
#endif
#undef NLG_CY_CHUNK
}

template <int DIM, bool KW, int BWC>
__global__ void __launch_bounds__(32 * cy_warps<DIM>(), DIM == 2 ? NLG_CY_MINB2 : NLG_CY_MINB3)
    stencil_cy_kernel(const __grid_constant__ CUtensorMap tmu, const __grid_constant__ CUtensorMap tmk, StArgs a) {
  constexpr int NWP = cy_warps<DIM>(), NT = 32 * NWP, TY = NWP * kCyR;
  extern __shared__ __align__(128) double csm[];
  __shared__ __align__(8) unsigned long long mbar[2];
  __shared__ int s_bmax;
  const Geom& g = a.g;
  const int H = a.H, hs = a.hs, BW = BWC ? BWC : cy_bw(hs), BHl = cy_bhl(hs, NWP), BOX = cy_box(hs, NWP);
  double* Tu = csm;
  double* Tk = KW ? csm + BOX : csm;
  const int MBOX = cy_mbox(hs, NWP), hx = cy_hx(hs);
  double* Mu = csm + (KW ? 2 : 1) * BOX;                 // 3-D mirror planes
  double* Mk = KW ? Mu + MBOX : Mu;
  const int W1 = H + 1, wfull = W1 * a.ws;               // table rows of one |dz|: [|dx|][dy + H]
  const int wlen = (hs + 1) * a.ws;                       // rows |dx| <= hs are all a sweep reads
  double* wt = Mu + (DIM == 3 ? (KW ? 2 : 1) * MBOX : 0);   // (rewritten per |dz| behind the tile barrier)
  int* isq = reinterpret_cast<int*>(wt + wlen);
  const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
  const int64_t n = g.n;
  int64_t x0, y0, z = 0;
  if (DIM == 2) {
    x0 = static_cast<int64_t>(blockIdx.x) * 32;
    y0 = g.row_begin + static_cast<int64_t>(blockIdx.y) * TY;
  } else {
    const int64_t ntx = (n + 31) / 32;
    z = g.row_begin + blockIdx.x;
    x0 = (blockIdx.y % ntx) * 32;
    y0 = (blockIdx.y / ntx) * TY;
  }
  const unsigned mb0 = static_cast<unsigned>(__cvta_generic_to_shared(mbar));
  const unsigned sTu = static_cast<unsigned>(__cvta_generic_to_shared(Tu));
  const unsigned sMu = static_cast<unsigned>(__cvta_generic_to_shared(Mu));
  const unsigned BYTES = static_cast<unsigned>(sizeof(double)) * BW * BHl * (KW ? 2 : 1);
  // boxes of one plane (u and kappa) -> dst, dst + box stride, completing on mbar[which]
  auto issue = [&](unsigned dst, int which, int64_t gz) {
    const unsigned mb = mb0 + 8u * which;
    const unsigned BOXB = static_cast<unsigned>(sizeof(double)) * (which ? MBOX : BOX);
    const int cx = static_cast<int>(x0) - hx;
    const int cy = static_cast<int>(DIM == 2 ? y0 - hs - g.in_begin : y0 - hs);
    const int cz = DIM == 2 ? 0 : static_cast<int>(gz - g.in_begin);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(BYTES) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(&tmu), "r"(cx), "r"(cy), "r"(cz), "r"(mb)
        : "memory");
    if (KW)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst + BOXB),
          "l"(&tmk), "r"(cx), "r"(cy), "r"(cz), "r"(mb)
          : "memory");
  };
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue(sTu, 0, z);
    s_bmax = -1;
  }
  for (int i = tid; i < isq_len(H); i += NT) {
    int x = static_cast<int>(sqrtf(static_cast<float>(i)));
    while (x * x > i) --x;
    while ((x + 1) * (x + 1) <= i) ++x;
    isq[i] = x;
  }
  // the three pad rows below the loaded box are read by overshoot steps only (never used): keep them finite
  for (int i = tid; i < 3 * BW; i += NT) {
    Tu[BW * BHl + i] = 0.0;
    if (KW) Tk[BW * BHl + i] = 0.0;
  }
  const int64_t ystop = DIM == 2 ? g.row_end : n;
  const int64_t ix = x0 + lane;
  const int64_t iy0 = y0 + wy * kCyR;
  const double inv_h = 1.0 / g.h;
  auto in_index = [&](int64_t iy) {
    return DIM == 2 ? (iy - g.in_begin) * n + ix : ((z - g.in_begin) * n + iy) * n + ix;
  };
  int M[kCyR];
  unsigned tiem = 0;
  int Mx = -1, Mn = 1 << 20;
  // the epilogue's per-target operands into L2 now (one line per row and array, lanes 0 and 16)
#ifndef NLG_CY_NOPF
  if ((lane & 15) == 0 && ix < n) {
    const int64_t shift = (g.row_begin - g.in_begin) * g.stride0;
#pragma unroll
    for (int r = 0; r < kCyR; ++r)
      if (iy0 + r < ystop) {
        const int64_t oi = in_index(iy0 + r) - shift;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.scale + oi));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.diag + oi));
      }
  }
#endif
#pragma unroll
  for (int r = 0; r < kCyR; ++r) {
    M[r] = -1;
    const int64_t iy = iy0 + r;
    if (ix < n && iy < ystop) {
      const double e = a.delta[in_index(iy)] * inv_h, e2 = e * e;
      const int mlo = static_cast<int>(ceil(e2 * (1.0 - tie_band_n(inv_h))));
      const int mhi = static_cast<int>(floor(e2 * (1.0 + tie_band_n(inv_h))));
      M[r] = mlo <= mhi ? mlo - 1 : mhi;
      if (mlo <= mhi) tiem |= 1u << r;
      Mn = min(Mn, M[r]);
    }
    Mx = max(Mx, M[r]);
  }
  const int MW = __reduce_max_sync(0xffffffffu, Mx);
  const int MN = __reduce_min_sync(0xffffffffu, Mn);
  __syncthreads();                                       // s_bmax, isq
  if (DIM == 3 && lane == 0) atomicMax(&s_bmax, MW);
  if (DIM == 3) __syncthreads();
  const int Rz = DIM == 3 ? (s_bmax < 0 ? -1 : isq[s_bmax]) : 0;
  if (DIM == 3 && tid == 0 && Rz >= 1) {
    issue(sMu, 1, z - 1);
  }
  if (Rz < 0) cy_mbar_wait(mb0, 0u);                     // (no live target: never leave a bulk copy in flight)
  double a0[kCyR], a1[kCyR];
#pragma unroll
  for (int r = 0; r < kCyR; ++r) a0[r] = a1[r] = 0.0;
  const int colbase = (wy * kCyR + hs) * BW + lane + hx;  // the lane's first target in the box
  for (int dz = 0; dz <= Rz; ++dz) {
    // weight rows of this |dz| (row dx = 0 halved: its column is added to itself)
    double* wd = wt;
    {
      const double* src = a.tab + static_cast<size_t>(dz) * wfull;
      for (int i = tid; i < wlen; i += NT) wd[i] = (i < a.ws ? 0.5 : 1.0) * __ldg(src + i);
    }
    cy_mbar_wait(mb0, static_cast<unsigned>(dz & 1));
    if (DIM == 3 && dz > 0) cy_mbar_wait(mb0 + 8u, static_cast<unsigned>((dz - 1) & 1));
    // combine: (u, kappa) [+ mirror] -> (u+ + u-, kappa+ u+ + kappa- u-)
    {
      double2* tu2 = reinterpret_cast<double2*>(Tu);
      double2* tk2 = reinterpret_cast<double2*>(Tk);
      const double2* mu2 = reinterpret_cast<const double2*>(Mu);
      const double2* mk2 = reinterpret_cast<const double2*>(Mk);
      const int ne2 = BW * BHl / 2;
      if (DIM == 3 && dz > 0) {
        for (int e = tid; e < ne2; e += NT) {
          double2 u = tu2[e];
          const double2 m = mu2[e];
          if (KW) {
            double2 k = tk2[e];
            const double2 km = mk2[e];
            k.x = fma(km.x, m.x, k.x * u.x);
            k.y = fma(km.y, m.y, k.y * u.y);
            tk2[e] = k;
          }
          u.x += m.x;
          u.y += m.y;
          tu2[e] = u;
        }
      } else if (KW) {
        for (int e = tid; e < ne2; e += NT) {
          const double2 u = tu2[e];
          double2 k = tk2[e];
          k.x *= u.x;
          k.y *= u.y;
          tk2[e] = k;
        }
      }
    }
    __syncthreads();                                     // tile + weights ready; mirror boxes consumed
    if (DIM == 3 && tid == 0 && dz + 1 <= Rz && dz >= 1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(sMu, 1, z - (dz + 1));
    }
    const int c00 = dz * dz;
    const int mW = MW - c00;
    if (mW >= 0) {
      const int XW = isq[mW];
      for (int dx = 0; dx <= XW; ++dx) {
        const int c0 = c00 + dx * dx;
        const int YW = isq[MW - c0];
#if NLG_CY_STEPSEL
        const int YN = MN <= MW ? MN : -1;
#else
        const int YN = MN >= c0 && MN <= MW ? isq[MN - c0] : -1;
#endif
        const int o = colbase - YW * BW;
        cy_sweep<KW, BWC, (DIM == 3 ? NLG_CY_U3 : NLG_CY_U)>(a0, a1, M, Tu + o + dx, Tu + o - dx, Tk + o + dx,
                                                              Tk + o - dx, BW, wd + dx * a.ws + H - YW, YW, YN, c0);
      }
    }
    if (DIM == 3 && dz + 1 <= Rz) {
      __syncthreads();                                   // the tile is consumed
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(sTu, 0, z + dz + 1);
      }
    }
  }
  // tie bands (rare): offsets with |d|^2 in [mlo, mhi] by the reference's float predicate, from global memory
  {
    unsigned tm = tiem;
    while (tm) {
      const int rr = __ffs(tm) - 1;
      tm &= tm - 1;
      const int64_t iy = iy0 + rr;
      const double delta = a.delta[in_index(iy)];
      const double e = delta * inv_h, e2 = e * e;
      const int mlo = static_cast<int>(ceil(e2 * (1.0 - tie_band_n(inv_h))));
      const int mhi = static_cast<int>(floor(e2 * (1.0 + tie_band_n(inv_h))));
      const int64_t ki[3] = {DIM == 2 ? iy : z, DIM == 2 ? ix : iy, ix};
      const int Rt = isqrt_floor(mhi);
      double t0 = 0.0, t1 = 0.0;
      for (int dz = (DIM == 3 ? -Rt : 0); dz <= (DIM == 3 ? Rt : 0); ++dz) {
        const int Ry = isqrt_floor(mhi - dz * dz);
        for (int dy = -Ry; dy <= Ry; ++dy) {
          const int X = isqrt_floor(mhi - dz * dz - dy * dy);
          const int m = dz * dz + dy * dy + X * X;
          if (m < mlo || m == 0) continue;
          for (int sx = -X; sx <= X; sx += (X > 0 ? 2 * X : 1)) {
            bool in;
            if (DIM == 2) {
              const int d[2] = {dy, sx};
              in = point_in<2>(ki, d, g.h, delta);
            } else {
              const int d[3] = {dz, dy, sx};
              in = point_in<3>(ki, d, g.h, delta);
            }
            if (!in) continue;
            const int64_t gz = z + dz, gy = iy + dy, gx = ix + sx;
            if (gy < 0 || gy >= n || gx < 0 || gx >= n) continue;
            if (DIM == 3 && (gz < 0 || gz >= n || gz < g.in_begin || gz >= g.in_end)) continue;
            if (DIM == 2 && (gy < g.in_begin || gy >= g.in_end)) continue;
            const int64_t k = DIM == 2 ? (gy - g.in_begin) * n + gx : ((gz - g.in_begin) * n + gy) * n + gx;
            const int az = dz < 0 ? -dz : dz, ay = dy < 0 ? -dy : dy;
            const double w = __ldg(a.tab + (static_cast<size_t>(DIM == 3 ? az : 0) * W1 + ay) * a.ws + sx + H);
            const double uu = a.u[k];
            t0 = fma(w, uu, t0);
            if (KW) t1 = fma(w, a.kappa[k] * uu, t1);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < kCyR; ++r) {
        if (r == rr) {
          a0[r] += t0;
          a1[r] += t1;
        }
      }
    }
  }
  if (ix >= n) return;
#pragma unroll
  for (int r = 0; r < kCyR; ++r) {
    const int64_t iy = iy0 + r;
    if (iy < ystop) {
      const int64_t ii = in_index(iy);
      const int64_t oi = ii - (g.row_begin - g.in_begin) * g.stride0;
      const double X = KW ? fma(a.kappa[ii], a0[r], a1[r]) : a0[r];
      a.out[oi] = a.scale[oi] * (X - a.u[ii] * a.diag[oi]);
    }
  }
}


// ---- column-lane apply, 2-D peridynamics (cfg3): stencil_cyp_kernel -----------
// Same blocking as stencil_cy_kernel. M(d) = d d^T / |d|^3: M00 and M11 are
// even in dx and M01 is odd, so the columns +dx / -dx enter as sums for the
// even entries and as differences for the odd one (half the FMAs of the
// row-lane sweep, which cannot pair):
//   out0 += M00 (u0+ + u0-) + M01 (u1+ - u1-),  out1 += M01 (u0+ - u0-) + M11 (u1+ + u1-),
// one output component per pass (two windows of kCyR + 4 in registers).
template <int PH, int BWC>
__device__ __forceinline__ void cyp_chunk(double (&acc)[kCyR], const int (&M)[kCyR], double (&Ws)[kCyR + kCyU],
                                          double (&Wd)[kCyR + kCyU], const double*& sp, const double*& sm,
                                          const double*& dp, const double*& dm, int bw_rt, const double*& wa,
                                          const double*& wb, int dy0, int YW, int YN, int c0) {
  constexpr int NW = kCyR + kCyU;
  const int BW = BWC ? BWC : bw_rt;
#pragma unroll
  for (int j = 0; j < kCyU; ++j) {
    Ws[(kCyR + j + kCyU * PH) % NW] = sp[j * BW] + sm[j * BW];
    Wd[(kCyR + j + kCyU * PH) % NW] = dp[j * BW] - dm[j * BW];
  }
  if (dy0 >= -YN && min(dy0 + kCyU - 1, YW) <= YN) {
#pragma unroll
    for (int s = 0; s < kCyU; ++s) {
      const bool on = dy0 + s <= YW;
      const double a = on ? wa[s] : 0.0, b = on ? wb[s] : 0.0;
#pragma unroll
      for (int r = 0; r < kCyR; ++r)
        acc[r] = fma(a, Ws[(s + r + kCyU * PH) % NW], fma(b, Wd[(s + r + kCyU * PH) % NW], acc[r]));
    }
  } else {
#pragma unroll
    for (int s = 0; s < kCyU; ++s) {
      const double a = wa[s], b = wb[s];
      const int c = c0 + (dy0 + s) * (dy0 + s);
#pragma unroll
      for (int r = 0; r < kCyR; ++r) {
        const double t = fma(a, Ws[(s + r + kCyU * PH) % NW], fma(b, Wd[(s + r + kCyU * PH) % NW], acc[r]));
        acc[r] = c <= M[r] ? t : acc[r];
      }
    }
  }
  sp += kCyU * BW;
  sm += kCyU * BW;
  dp += kCyU * BW;
  dm += kCyU * BW;
  wa += kCyU;
  wb += kCyU;
}

template <int BWC>
__device__ __forceinline__ void cyp_sweep(double (&acc)[kCyR], const int (&M)[kCyR], const double* sp,
                                          const double* sm, const double* dp, const double* dm, int bw_rt,
                                          const double* wa, const double* wb, int YW, int YN, int c0) {
  const int BW = BWC ? BWC : bw_rt;
  double Ws[kCyR + kCyU], Wd[kCyR + kCyU];
#pragma unroll
  for (int i = 0; i < kCyR; ++i) {
    Ws[i] = sp[i * BW] + sm[i * BW];
    Wd[i] = dp[i * BW] - dm[i * BW];
  }
  sp += kCyR * BW;
  sm += kCyR * BW;
  dp += kCyR * BW;
  dm += kCyR * BW;
  const int nsteps = 2 * YW + 1;
  int s0 = 0;
#define NLG_CYP_CHUNK(PH)                                                             \
  cyp_chunk<PH, BWC>(acc, M, Ws, Wd, sp, sm, dp, dm, BW, wa, wb, s0 - YW, YW, YN, c0);  \
  s0 += kCyU;                                                                         \
  if (s0 >= nsteps) break;
  for (;;) {
    NLG_CYP_CHUNK(0)
    NLG_CYP_CHUNK(1)
    NLG_CYP_CHUNK(2)
#if NLG_CY_NPH >= 4
    NLG_CYP_CHUNK(3)
#endif
#if NLG_CY_NPH >= 5
    NLG_CYP_CHUNK(4)
#endif
  }
#undef NLG_CYP_CHUNK
}

template <int BWC>
__global__ void __launch_bounds__(32 * NLG_CYP_W, NLG_CYP_MINB)
    stencil_cyp_kernel(const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1, StArgs a) {
  constexpr int NWP = NLG_CYP_W, NT = 32 * NWP, TY = NWP * kCyR;
  extern __shared__ __align__(128) double csm[];
  __shared__ __align__(8) unsigned long long mbar;
  const Geom& g = a.g;
  const int H = a.H, hs = a.hs, BW = BWC ? BWC : cy_bw(hs), BHl = cy_bhl(hs, NWP), BOX = cy_box(hs, NWP);
  double* U0 = csm;
  double* U1 = csm + BOX;
  const int W1 = H + 1, wlen = W1 * a.ws;                // rows dx = 0..H of one table: [dx][dy + H]
  double* wt = csm + 2 * BOX;                             // M11 | M01 | M00 of the table (= M00 | M01 | M11 transposed)
  int* isq = reinterpret_cast<int*>(wt + 3 * wlen);
  const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
  const int64_t n = g.n;
  const int64_t x0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int64_t y0 = g.row_begin + static_cast<int64_t>(blockIdx.y) * TY;
  const unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(&mbar));
  if (tid == 0) {
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(U0));
    const unsigned BYTES = static_cast<unsigned>(sizeof(double)) * BW * BHl * 2;
    const int cx = static_cast<int>(x0) - cy_hx(hs), cy = static_cast<int>(y0 - hs - g.in_begin);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(BYTES) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(&tm0), "r"(cx), "r"(cy), "r"(0), "r"(mb)
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            dst + static_cast<unsigned>(sizeof(double)) * BOX),
        "l"(&tm1), "r"(cx), "r"(cy), "r"(0), "r"(mb)
        : "memory");
  }
  for (int i = tid; i < isq_len(H); i += NT) {
    int x = static_cast<int>(sqrtf(static_cast<float>(i)));
    while (x * x > i) --x;
    while ((x + 1) * (x + 1) <= i) ++x;
    isq[i] = x;
  }
  for (int i = tid; i < 3 * BW; i += NT) {
    U0[BW * BHl + i] = 0.0;
    U1[BW * BHl + i] = 0.0;
  }
  // table rows dx >= 0 (row H + dx of the signed table); the dx = 0 rows halved (their column is added to itself)
  for (int i = tid; i < 3 * wlen; i += NT) {
    const int t = i / wlen, k = i - t * wlen;
    wt[i] = (k < a.ws ? 0.5 : 1.0) * __ldg(a.tab + static_cast<size_t>(t) * a.wp + static_cast<size_t>(H) * a.ws + k);
  }
  const int64_t ystop = g.row_end;
  const int64_t ix = x0 + lane;
  const int64_t iy0 = y0 + wy * kCyR;
  const double inv_h = 1.0 / g.h;
  const int64_t nin_total = (g.in_end - g.in_begin) * g.stride0;
  const int64_t plane_out = a.plane_out;
  auto in_index = [&](int64_t iy) { return (iy - g.in_begin) * n + ix; };
  int M[kCyR];
  unsigned tiem = 0;
  int Mx = -1, Mn = 1 << 20;
  if ((lane & 15) == 0 && ix < n) {
    const int64_t shift = (g.row_begin - g.in_begin) * g.stride0;
#pragma unroll
    for (int r = 0; r < kCyR; ++r)
      if (iy0 + r < ystop) {
        const int64_t oi = in_index(iy0 + r) - shift;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.scale + oi));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.diag + oi));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.diag + plane_out + oi));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.diag + 2 * plane_out + oi));
      }
  }
#pragma unroll
  for (int r = 0; r < kCyR; ++r) {
    M[r] = -1;
    const int64_t iy = iy0 + r;
    if (ix < n && iy < ystop) {
      const double e = a.delta[in_index(iy)] * inv_h, e2 = e * e;
      const int mlo = static_cast<int>(ceil(e2 * (1.0 - tie_band_n(inv_h))));
      const int mhi = static_cast<int>(floor(e2 * (1.0 + tie_band_n(inv_h))));
      M[r] = mlo <= mhi ? mlo - 1 : mhi;
      if (mlo <= mhi) tiem |= 1u << r;
      Mn = min(Mn, M[r]);
    }
    Mx = max(Mx, M[r]);
  }
  const int MW = __reduce_max_sync(0xffffffffu, Mx);
  const int MN = __reduce_min_sync(0xffffffffu, Mn);
  double a0[kCyR], a1[kCyR];
#pragma unroll
  for (int r = 0; r < kCyR; ++r) a0[r] = a1[r] = 0.0;
  __syncthreads();                                       // tables
  cy_mbar_wait(mb, 0u);
  const int colbase = (wy * kCyR + hs) * BW + lane + cy_hx(hs);
  if (MW >= 0) {
    const int XW = isq[MW];
    const double* w11 = wt;                               // table 0: dy'^2 / r^3 read transposed = M11(dy, dx)... see below
    const double* w01 = wt + wlen;
    const double* w00 = wt + 2 * wlen;
    // the table stores t0 = dy^2/r^3, t1 = dx dy/r^3, t2 = dx^2/r^3 at [dy + H][dx + H]; read at
    // [dx + H][dy + H] they are M11, M01, M00 of the offset (dy, dx)
    for (int dx = 0; dx <= XW; ++dx) {
      const int c0 = dx * dx;
      const int YW = isq[MW - c0];
      const int YN = MN >= c0 && MN <= MW ? isq[MN - c0] : -1;
      const int o = colbase - YW * BW, wo = dx * a.ws + H - YW;
      // one inlined sweep for both output components: pass 0 sums into a0 (even entry M00 on u0, odd on u1),
      // pass 1 into a1 (M11 on u1, odd on u0); the accumulator arrays trade places after each pass
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        const double* S = pass ? U1 : U0;
        const double* D = pass ? U0 : U1;
        cyp_sweep<BWC>(a0, M, S + o + dx, S + o - dx, D + o + dx, D + o - dx, BW, (pass ? w11 : w00) + wo, w01 + wo, YW,
                       YN, c0);
#pragma unroll
        for (int r = 0; r < kCyR; ++r) {
          const double t = a0[r];
          a0[r] = a1[r];
          a1[r] = t;
        }
      }
    }
  }
  // tie bands (rare): from global memory with the reference's float predicate
  {
    unsigned tm = tiem;
    while (tm) {
      const int rr = __ffs(tm) - 1;
      tm &= tm - 1;
      const int64_t iy = iy0 + rr;
      const double delta = a.delta[in_index(iy)];
      const double e = delta * inv_h, e2 = e * e;
      const int mlo = static_cast<int>(ceil(e2 * (1.0 - tie_band_n(inv_h))));
      const int mhi = static_cast<int>(floor(e2 * (1.0 + tie_band_n(inv_h))));
      const int64_t ki[3] = {iy, ix, 0};
      const int Ry = isqrt_floor(mhi);
      double t0 = 0.0, t1 = 0.0;
      for (int dy = -Ry; dy <= Ry; ++dy) {
        const int X = isqrt_floor(mhi - dy * dy);
        const int m = dy * dy + X * X;
        if (m < mlo || m == 0) continue;
        for (int sx = -X; sx <= X; sx += (X > 0 ? 2 * X : 1)) {
          const int d[2] = {dy, sx};
          if (!point_in<2>(ki, d, g.h, delta)) continue;
          const int64_t gy = iy + dy, gx = ix + sx;
          if (gy < 0 || gy >= n || gx < 0 || gx >= n || gy < g.in_begin || gy >= g.in_end) continue;
          const int64_t k = (gy - g.in_begin) * n + gx;
          const int t = (dy + H) * a.ws + sx + H;
          const double mxx = __ldg(a.tab + t), mxy = __ldg(a.tab + a.wp + t), myy = __ldg(a.tab + 2 * a.wp + t);
          const double vx = a.u[k], vy = a.u[nin_total + k];
          t0 = fma(mxx, vx, fma(mxy, vy, t0));
          t1 = fma(mxy, vx, fma(myy, vy, t1));
        }
      }
#pragma unroll
      for (int r = 0; r < kCyR; ++r) {
        if (r == rr) {
          a0[r] += t0;
          a1[r] += t1;
        }
      }
    }
  }
  if (ix >= n) return;
#pragma unroll
  for (int r = 0; r < kCyR; ++r) {
    const int64_t iy = iy0 + r;
    if (iy < ystop) {
      const int64_t ii = in_index(iy);
      const int64_t oi = ii - (g.row_begin - g.in_begin) * g.stride0;
      const double ux = a.u[ii], uy = a.u[nin_total + ii];
      const double dxx = a.diag[oi], dxy = a.diag[plane_out + oi], dyy = a.diag[2 * plane_out + oi];
      const double sc = a.scale[oi];
      a.out[oi] = sc * (a0[r] - (dxx * ux + dxy * uy));
      a.out[plane_out + oi] = sc * (a1[r] - (dxy * ux + dyy * uy));
    }
  }
}

// 1-D fractional apply (horizons below the scan threshold, e.g. cfg0): S
// lanes per target over a shared-memory tile of the CTA's neighbourhood, lane
// s summing the offsets k = s mod S of the target's span, then a shuffle
// reduction. S = 8 when one target per thread would leave most SMs idle
// (cfg0: 4096 targets = 16 CTAs of 256; with S = 8, 128 CTAs of 32 targets).
constexpr int k1T = 256;

template <bool KW, int S>
__global__ void __launch_bounds__(k1T) stencil1d_kernel(StArgs a) {
  extern __shared__ double sm[];
  constexpr int TPC = k1T / S;                         // targets per CTA
  const int H = a.H;
  const int TW = TPC + 2 * H;
  double2* tile = reinterpret_cast<double2*>(sm);
  double* wt = sm + 2 * static_cast<size_t>(TW);
  for (int i = threadIdx.x; i < a.tab_len; i += k1T) wt[i] = a.tab[i];
  const Geom& g = a.g;
  const int64_t n = g.n;
  const int64_t x0 = g.row_begin + static_cast<int64_t>(blockIdx.x) * TPC;
  for (int i = threadIdx.x; i < TW; i += k1T) {
    const int64_t gx = x0 - H + i;
    const bool in = gx >= 0 && gx < n && gx >= g.in_begin && gx < g.in_end;
    const int64_t k = gx - g.in_begin;
    double2 v = make_double2(0.0, 0.0);
    if (in) {
      if (KW) v = a.pk[k];
      else v.x = __ldg(a.u + k);
    }
    tile[i] = v;
  }
  __syncthreads();
  const int t = threadIdx.x / S, ls = threadIdx.x % S;  // target within the CTA, lane within its group
  const int64_t ix = x0 + t;
  const bool live = ix < g.row_end;
  const int64_t ii = ix - g.in_begin;
  double acc0 = 0.0, acc1 = 0.0;
  const double2* trow = tile + t + H;
  if (live) {
    Ball<1> B;
    B.init(a.delta ? a.delta[ii] : a.delta0, g.h);
    B.ki[0] = ix;
    int d[1] = {0};
    int xm, xp;
    if (B.span(d, xm, xp)) {
      if (S == 1) {
        row_sum<KW>(trow, wt + H, xm, xp, acc0, acc1);
      } else {
        const double* w = wt + H;
        for (int k = -xm + ls; k <= xp; k += S) {
          const double2 v = trow[k];
          acc0 = fma(w[k], v.x, acc0);
          if (KW) acc1 = fma(w[k], v.y, acc1);
        }
      }
    }
  }
  if (S > 1) {   // groups of S consecutive lanes (S divides 32)
#pragma unroll
    for (int o = S / 2; o > 0; o >>= 1) {
      acc0 += __shfl_xor_sync(0xffffffffu, acc0, o);
      if (KW) acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
    }
  }
  if (!live || ls != 0) return;
  const int64_t oi = ix - g.row_begin;
  const double X = KW ? fma(a.kappa[ii], acc0, acc1) : acc0;
  a.out[oi] = a.scale[oi] * (X - trow[0].x * a.diag[oi]);
}

__global__ void pack_kernel(const double* u, const double* kappa, int64_t n, double2* pk) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    const double v = u[i];
    pk[i] = make_double2(v, v * kappa[i]);
  }
}


template <int DIM, int KIND, int MODE, bool KW>
void launch_t(const StArgs& a, cudaStream_t s, size_t smem) {
  const int64_t n = a.g.n;
  const int64_t nx = DIM == 1 ? (a.g.row_end - a.g.row_begin) : n;
  const int64_t rows = DIM == 1 ? 1 : (a.g.row_end - a.g.row_begin) * (DIM == 3 ? n : 1);
  const int64_t bx = (nx + kTX - 1) / kTX, by = (rows + kTY - 1) / kTY;
  stencil_kernel<DIM, KIND, MODE, KW><<<static_cast<unsigned>(bx * by), dim3(kTX, kTY), smem, s>>>(a);
}

size_t tile2d_bytes(const StArgs& a) {
  const size_t wlen = a.g.dim == 2 ? a.tab_len : static_cast<size_t>(a.H + 1) * a.ws;
  return sizeof(double2) * static_cast<size_t>(kBY + 2 * a.H + 1) * tile2d_rs(a.H, tile_bx_rt(a.g.dim, a.kind)) +
         sizeof(double) * wlen +
         sizeof(int) * (isq_len(a.H) + 1);
}

void launch(const StArgs& a, cudaStream_t s, size_t smem) {
  const int dim = a.g.dim;
  const int64_t n = a.g.n;
  if (dim == 1) {
    if (a.mode == 0) {
      const int64_t nt = a.g.row_end - a.g.row_begin;
      const bool split = (nt + k1T - 1) / k1T < 2 * 148;   // too few CTAs for one target per thread
      const int tpc = split ? k1T / 8 : k1T;
      const unsigned grid = static_cast<unsigned>((nt + tpc - 1) / tpc);
      const size_t sb = sizeof(double) * (2 * static_cast<size_t>(tpc + 2 * a.H) + a.tab_len);
      if (split) {
        if (a.kw) stencil1d_kernel<true, 8><<<grid, k1T, sb, s>>>(a);
        else stencil1d_kernel<false, 8><<<grid, k1T, sb, s>>>(a);
      } else {
        if (a.kw) stencil1d_kernel<true, 1><<<grid, k1T, sb, s>>>(a);
        else stencil1d_kernel<false, 1><<<grid, k1T, sb, s>>>(a);
      }
    } else {
      if (a.kw) launch_t<1, 0, 1, true>(a, s, smem); else launch_t<1, 0, 1, false>(a, s, smem);
    }
    return;
  }
  if (dim == 2 && a.mode == 0) {
    const int bx = tile_bx_rt(2, a.kind);
    dim3 grid(static_cast<unsigned>((n + bx - 1) / bx),
              static_cast<unsigned>((a.g.row_end - a.g.row_begin + kBY - 1) / kBY));
    const size_t sb = tile2d_bytes(a);
    constexpr int kWF = tile_bx<2, 0>() / kR2Frac, kWP = tile_bx<2, 1>() / kR2Peri;   // warps per CTA
    if (a.kind == 1) stencil_rb_kernel<2, 1, false, kR2Peri><<<grid, dim3(32, kWP), sb, s>>>(a);
    else if (a.kw) stencil_rb_kernel<2, 0, true, kR2Frac><<<grid, dim3(32, kWF), sb, s>>>(a);
    else stencil_rb_kernel<2, 0, false, kR2Frac><<<grid, dim3(32, kWF), sb, s>>>(a);
    return;
  }
  if (dim == 3 && a.mode == 0) {
    constexpr int bx = tile_bx<3, 0>(), kW3 = bx / kR3Frac;
    const int64_t ntx = (n + bx - 1) / bx, nty = (n + kBY - 1) / kBY;
    dim3 grid(static_cast<unsigned>(a.g.row_end - a.g.row_begin), static_cast<unsigned>(ntx * nty));
    const size_t sb = tile2d_bytes(a);
    if (a.kw) stencil_rb_kernel<3, 0, true, kR3Frac><<<grid, dim3(32, kW3), sb, s>>>(a);
    else stencil_rb_kernel<3, 0, false, kR3Frac><<<grid, dim3(32, kW3), sb, s>>>(a);
    return;
  }
  if (a.kind == 1) {
    if (a.mode == 0) launch_t<2, 1, 0, false>(a, s, smem);
    else launch_t<2, 1, 1, false>(a, s, smem);
    return;
  }
  if (dim == 2) {
    if (a.mode == 0) { if (a.kw) launch_t<2, 0, 0, true>(a, s, smem); else launch_t<2, 0, 0, false>(a, s, smem); }
    else { if (a.kw) launch_t<2, 0, 1, true>(a, s, smem); else launch_t<2, 0, 1, false>(a, s, smem); }
  } else {
    if (a.mode == 0) { if (a.kw) launch_t<3, 0, 0, true>(a, s, smem); else launch_t<3, 0, 0, false>(a, s, smem); }
    else { if (a.kw) launch_t<3, 0, 1, true>(a, s, smem); else launch_t<3, 0, 1, false>(a, s, smem); }
  }
}


// Tensor map over an input field for the column-lane apply: (x: n, y: n or the
// input rows, z: input planes or 1), boxes of (32 + 2 hs) x (rows + 2 hs) x 1,
// zero fill outside.
bool cy_encode(CUtensorMap* m, const double* base, int dim, int64_t n, int64_t rows_in, int hs, int warps) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess || !fn)
      return false;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if ((n * 8) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(dim == 2 ? rows_in : n),
                              static_cast<cuuint64_t>(dim == 2 ? 1 : rows_in)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(n) * 8, static_cast<cuuint64_t>(n) * dims[1] * 8};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(cy_bw(hs)), static_cast<cuuint32_t>(cy_bhl(hs, warps)), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t cy_smem(const StArgs& a, int dim) {
  const int warps = cy_warps_rt(dim, a.kind);
  const int nf = a.kind == 1 ? 2 : (a.kw ? 2 : 1);
  const size_t wlen = a.kind == 1 ? static_cast<size_t>(a.H + 1) * a.ws * 3 : static_cast<size_t>(a.hs + 1) * a.ws;
  return sizeof(double) * (static_cast<size_t>(nf) * (cy_box(a.hs, warps) + (dim == 3 ? cy_mbox(a.hs, warps) : 0)) + wlen) +
         sizeof(int) * (isq_len(a.H) + 1);
}

// the column-lane launch; false when the tensor map of u cannot be encoded (the caller falls back)
bool launch_cy(StencilState& S, const StArgs& a, cudaStream_t s) {
  const int dim = a.g.dim;
  const int64_t n = a.g.n, rows_in = a.g.in_end - a.g.in_begin;
  const int warps = cy_warps_rt(dim, a.kind);
  if (S.tmu_base != a.u) {
    if (!cy_encode(&S.tmu, a.u, dim, n, rows_in, S.hs, warps)) return false;
    if (a.kind == 1 && !cy_encode(&S.tmu1, a.u + rows_in * a.g.stride0, dim, n, rows_in, S.hs, warps)) return false;
    S.tmu_base = a.u;
  }
  const size_t sb = cy_smem(a, dim);
  const int bw = cy_bw(S.hs);
  if (a.kind == 1) {
    dim3 grid(static_cast<unsigned>((n + 31) / 32),
              static_cast<unsigned>((a.g.row_end - a.g.row_begin + warps * kCyR - 1) / (warps * kCyR)));
    if (bw == kCyBWp) stencil_cyp_kernel<kCyBWp><<<grid, 32 * warps, sb, s>>>(S.tmu, S.tmu1, a);
    else stencil_cyp_kernel<0><<<grid, 32 * warps, sb, s>>>(S.tmu, S.tmu1, a);
    return true;
  }
  if (dim == 2) {
    dim3 grid(static_cast<unsigned>((n + 31) / 32),
              static_cast<unsigned>((a.g.row_end - a.g.row_begin + warps * kCyR - 1) / (warps * kCyR)));
    if (bw == kCyBW2) {
      if (a.kw) stencil_cy_kernel<2, true, kCyBW2><<<grid, 32 * warps, sb, s>>>(S.tmu, S.tmk, a);
      else stencil_cy_kernel<2, false, kCyBW2><<<grid, 32 * warps, sb, s>>>(S.tmu, S.tmu, a);
    } else {
      if (a.kw) stencil_cy_kernel<2, true, 0><<<grid, 32 * warps, sb, s>>>(S.tmu, S.tmk, a);
      else stencil_cy_kernel<2, false, 0><<<grid, 32 * warps, sb, s>>>(S.tmu, S.tmu, a);
    }
  } else {
    const int64_t ntx = (n + 31) / 32, nty = (n + warps * kCyR - 1) / (warps * kCyR);
    dim3 grid(static_cast<unsigned>(a.g.row_end - a.g.row_begin), static_cast<unsigned>(ntx * nty));
    if (bw == kCyBW3) {
      if (a.kw) stencil_cy_kernel<3, true, kCyBW3><<<grid, 32 * warps, sb, s>>>(S.tmu, S.tmk, a);
      else stencil_cy_kernel<3, false, kCyBW3><<<grid, 32 * warps, sb, s>>>(S.tmu, S.tmu, a);
    } else {
      if (a.kw) stencil_cy_kernel<3, true, 0><<<grid, 32 * warps, sb, s>>>(S.tmu, S.tmk, a);
      else stencil_cy_kernel<3, false, 0><<<grid, 32 * warps, sb, s>>>(S.tmu, S.tmu, a);
    }
  }
  return true;
}

StArgs make_args(const Plan& P, const StencilState& S, int mode, const double* u, double* out) {
  StArgs a;
  a.g = P.geom;
  a.kind = S.kind;
  a.kw = P.d_kappa != nullptr && S.kind == 0;
  a.collar = P.exterior == 1;
  a.mode = mode;
  a.H = S.H;
  a.hs = S.hs;
  a.plane_out = P.n_out;
  a.u = u;
  a.pk = reinterpret_cast<const double2*>(S.pack);
  a.delta = P.d_delta;
  a.delta0 = P.delta0;
  a.kappa = P.d_kappa;
  a.tab = S.kind == 0 ? S.wtab : S.mtab;
  a.tab_len = static_cast<int>(S.tab_bytes / sizeof(double));
  a.ws = S.ws;
  a.wp = (2 * S.H + 1) * S.ws;
  a.diag = S.diag;
  a.scale = S.scale;
  a.out = out;
  return a;
}

}  // namespace

namespace {
template <typename K>
void smem_attr(K k) {
  NLG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  NLG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
}
void allow_smem() {
  smem_attr(stencil_rb_kernel<2, 0, true, kR2Frac>);
  smem_attr(stencil_rb_kernel<2, 0, false, kR2Frac>);
  smem_attr(stencil_rb_kernel<2, 1, false, kR2Peri>);
  smem_attr(stencil_rb_kernel<3, 0, true, kR3Frac>);
  smem_attr(stencil_rb_kernel<3, 0, false, kR3Frac>);
  smem_attr(stencil_cy_kernel<2, true, 0>);
  smem_attr(stencil_cy_kernel<2, false, 0>);
  smem_attr(stencil_cy_kernel<3, true, 0>);
  smem_attr(stencil_cy_kernel<3, false, 0>);
  smem_attr(stencil_cy_kernel<2, true, kCyBW2>);
  smem_attr(stencil_cy_kernel<2, false, kCyBW2>);
  smem_attr(stencil_cy_kernel<3, true, kCyBW3>);
  smem_attr(stencil_cy_kernel<3, false, kCyBW3>);
  smem_attr(stencil_cyp_kernel<0>);
  smem_attr(stencil_cyp_kernel<kCyBWp>);
  smem_attr(stencil1d_kernel<true, 1>);
  smem_attr(stencil1d_kernel<false, 1>);
  smem_attr(stencil1d_kernel<true, 8>);
  smem_attr(stencil1d_kernel<false, 8>);
  smem_attr(stencil_kernel<1, 0, 1, true>);
  smem_attr(stencil_kernel<1, 0, 1, false>);
  smem_attr(stencil_kernel<2, 0, 0, true>);
  smem_attr(stencil_kernel<2, 0, 0, false>);
  smem_attr(stencil_kernel<2, 0, 1, true>);
  smem_attr(stencil_kernel<2, 0, 1, false>);
  smem_attr(stencil_kernel<2, 1, 0, false>);
  smem_attr(stencil_kernel<2, 1, 1, false>);
  smem_attr(stencil_kernel<3, 0, 0, true>);
  smem_attr(stencil_kernel<3, 0, 0, false>);
  smem_attr(stencil_kernel<3, 0, 1, true>);
  smem_attr(stencil_kernel<3, 0, 1, false>);
}
}  // namespace

// Method 3 applies when the operator is a BASELINE kernel in 2-D/3-D with a
// horizon of at most 16 cells (tables in shared memory).
void stencil_setup(Plan& P, const nlg_desc& d) {
  const Geom& g = P.geom;
  const bool frac = d.family == NLG_FRACTIONAL, peri = d.family == NLG_PERIDYNAMIC;
  if (!frac && !(peri && g.dim == 2)) return;
  // tile halo: every included offset has |d_a| <= floor(delta_max / h (1 + 1e-12)) <= floor(delta_max / h) + 1
#ifndef NLG_ST_HPAD
#define NLG_ST_HPAD 1
#endif
  const int H = static_cast<int>(std::floor(P.delta_max / g.h)) + NLG_ST_HPAD;
  if (g.dim >= 2 && H > 16) return;
  if (g.dim == 1 && H > 2048) return;
  auto* S = new StencilState();
  S->dim = g.dim;
  S->kind = peri ? 1 : 0;
  S->H = H;
  // 2-D / 3-D rows are read up to index 2H+11 by the register-blocked sweep
  S->ws = g.dim >= 2 ? ((2 * H + 12 + 3) & ~3) : 2 * H + 1;
  if (frac) {
    // symmetric rows: w[(az * W1 + ay) * W2 + dx + H] = |(az, ay, dx)|^-alpha, w = 0 at the origin
    const int W1 = H + 1, W2 = S->ws;
    const int nz = g.dim == 3 ? W1 : 1, ny = g.dim >= 2 ? W1 : 1;
    std::vector<double> w(static_cast<size_t>(nz) * ny * W2, 0.0);
    for (int az = 0; az < nz; ++az)
      for (int ay = 0; ay < ny; ++ay)
        for (int dx = -H; dx <= H; ++dx) {
          const int m = az * az + ay * ay + dx * dx;
          if (m == 0) continue;
          w[(static_cast<size_t>(az) * ny + ay) * W2 + dx + H] = std::pow(static_cast<double>(m), -0.5 * d.alpha);
        }
    S->wtab = upload_on(w, P.stream);
    S->tab_bytes = w.size() * sizeof(double);
  } else {
    const int W2 = S->ws, TP = (2 * H + 1) * W2;
    std::vector<double> t(static_cast<size_t>(3 * TP), 0.0);
    for (int dy = -H; dy <= H; ++dy)
      for (int dx = -H; dx <= H; ++dx) {
        const double r2 = static_cast<double>(dx * dx + dy * dy);
        if (r2 == 0.0) continue;
        const double r3 = r2 * std::sqrt(r2);
        const int k = (dy + H) * W2 + (dx + H);
        t[k] = dy * dy / r3;                 // axis 0 = "x" component of the SoA planes
        t[TP + k] = dx * dy / r3;
        t[2 * TP + k] = dx * dx / r3;
      }
    S->mtab = upload_on(t, P.stream);
    S->tab_bytes = t.size() * sizeof(double);
  }
  // s_i: fractional h^{d-alpha} C_i (x 1/2 with kappa); peridynamic -h^{d-1} c_i
  std::vector<double> sc(P.n_out);
  const double hd = g.hd;
  // the node-independent factor once (same operation order as factor * c per node)
  const double f = frac ? (d.kappa ? 0.5 : 1.0) * hd * std::pow(g.h, -d.alpha) : -hd / g.h;
  for (int64_t i = 0; i < P.n_out; ++i) {
    const int64_t x = P.halo_lo * g.stride0 + i;
    sc[i] = f * (d.coeff ? d.coeff[x] : d.coeff0);
  }
  S->scale = upload_on(sc, P.stream);
  S->scale_const = d.coeff == nullptr;
  S->scale0 = sc.empty() ? 0.0 : sc[0];
  NLG_CUDA(cudaMalloc(&S->diag, sizeof(double) * P.n_out * (peri ? 3 : 1)));
  if (frac && d.kappa && g.dim == 1) NLG_CUDA(cudaMalloc(&S->pack, sizeof(double2) * P.n_in));
  P.st_state = S;
  allow_smem();
  // diag: MODE 1 over the same sets and tables
  const StArgs a = make_args(P, *S, 1, nullptr, S->diag);
  launch(a, P.stream, S->tab_bytes);
  NLG_CUDA(cudaGetLastError());
  NLG_CUDA(cudaStreamSynchronize(P.stream));
  if (frac && g.dim == 3) S->box = boxfft_setup(P, d.alpha);
  // column-lane apply: per-node horizons in 2-D / 3-D (NLG_ST_CY=0 keeps the row-lane sweep)
  {   // the largest |d|^2 any target can include (its tie band counted), with a margin on the host rounding
    const double e = P.delta_max / g.h, m = std::floor(e * e * (1.0 + tie_band(g.h)) * (1.0 + 1e-9));
    int r = static_cast<int>(std::sqrt(m));
    while (static_cast<double>(r) * r > m) --r;
    while (static_cast<double>(r + 1) * (r + 1) <= m) ++r;
    S->hs = std::min(H, r);
#ifdef NLG_CY_HSOLD
    S->hs = H;
#endif
  }
  if ((frac || peri) && g.dim >= 2 && P.d_delta && !S->box) {
    const char* ce = std::getenv("NLG_ST_CY");
    const int warps = cy_warps_rt(g.dim, S->kind);
    StArgs t = make_args(P, *S, 0, nullptr, nullptr);
    S->cy = !(ce && std::atoi(ce) == 0) && cy_smem(t, g.dim) <= 200 * 1024 &&
            (!P.d_kappa || cy_encode(&S->tmk, P.d_kappa, g.dim, g.n, g.in_end - g.in_begin, S->hs, warps)) &&
            (g.n * 8) % 16 == 0;
  }
  P.fast_method = 3;
}

int stencil_launches(const Plan& P) {
  const StencilState* S = P.st_state;
  if (S->box) return boxfft_launches(*S->box);
  return S->pack ? 2 : 1;
}

bool stencil_box(const Plan& P) { return P.st_state && P.st_state->box; }

int stencil_fft_len(const Plan& P) { return P.st_state && P.st_state->box ? boxfft_length(*P.st_state->box) : 0; }

void stencil_apply(Plan& P, const double* u, double* out, cudaStream_t s) {
  StencilState* S = P.st_state;
  if (S->box) {
    boxfft_apply(P, *S->box, u, S->scale_const ? nullptr : S->scale, S->scale0, S->diag, out, s);
    return;
  }
  if (S->pack) {
    pack_kernel<<<static_cast<unsigned>((P.n_in + 255) / 256), 256, 0, s>>>(
        u, P.d_kappa, P.n_in, reinterpret_cast<double2*>(S->pack));
  }
  const StArgs a = make_args(P, *S, 0, u, out);
  if (S->cy && launch_cy(*S, a, s)) return;
  launch(a, s, S->tab_bytes);
}

// Row-range pieces of the apply (the chunked host pipeline of nlg_apply_fast).
// Output rows [a, b) relative to row_begin; u covers the plan's input rows
// (peridynamics: the component planes of u / out / diag stay strided by the
// plan's n_in / n_out).
void stencil_apply_rows(Plan& P, const double* u, double* out, int64_t a, int64_t b, cudaStream_t s) {
  StencilState* S = P.st_state;
  if (b <= a) return;
  const int64_t off = a * P.geom.stride0;
  StArgs A = make_args(P, *S, 0, u, out + off);
  A.g.row_begin = P.geom.row_begin + a;
  A.g.row_end = P.geom.row_begin + b;
  A.diag = S->diag + off;
  A.scale = S->scale ? S->scale + off : nullptr;
  if (S->cy && launch_cy(*S, A, s)) return;
  launch(A, s, S->tab_bytes);
}
void stencil_box_in(Plan& P, const double* u, int64_t p0, int64_t p1, cudaStream_t s) {
  boxfft_in(P, *P.st_state->box, u, p0, p1, s);
}
void stencil_box_out(Plan& P, const double* u, double* out, int64_t q0, int64_t q1, cudaStream_t s) {
  StencilState* S = P.st_state;
  boxfft_out(P, *S->box, u, S->scale_const ? nullptr : S->scale, S->scale0, S->diag, out, q0, q1, s);
}
int stencil_reach_rows(const Plan& P) { return P.st_state ? P.st_state->H : 0; }
// output rows per CTA row of the sweep: row ranges cut at multiples of it keep
// the CTA tiling (and so every warp's sweep range and summation order) of the
// one-call apply, so a chunked apply is bit-identical to it
int stencil_row_tile(const Plan& P) {
  if (P.geom.dim != 2) return 1;
  return P.st_state && P.st_state->cy ? std::max(kBY, cy_warps<2>() * kCyR) : kBY;
}
int stencil_components(const Plan& P) { return P.st_state ? (P.st_state->kind == 1 ? P.geom.dim : 1) : 1; }

void stencil_free(Plan& P) {
  StencilState* S = P.st_state;
  if (!S) return;
  for (double* p : {S->wtab, S->mtab, S->diag, S->scale, S->pack}) cudaFree(p);
  boxfft_free(S->box);
  delete S;
  P.st_state = nullptr;
}

}  // namespace nlg
