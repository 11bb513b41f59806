// paper_1905_08375_b200/csrc/spans.cu — fast method 1: polynomial-truncated
// K = 0 operator (the reference's TruncatedOperator for d = 1..3) by row
// prefix sums and span differences.
//
// Reference semantics (operators.cpp:126-167, tree.cpp:35-58,115-161): the
// Algorithm-1 panels of node x cover exactly the Leaf-rule node set
// (test_tree.cpp:99-115), which is convex along every grid row. So
//   S_i = sum_{panels} M_0(panel) = sum_{rows r of the ball} (P_r(b+1) - P_r(a))
// with P_r the prefix sum of u along the fastest axis and [a,b] the exact
// Leaf (or Point) span of row r. Prefix sums are compensated (double-double)
// and restarted per 1024-node segment, so |prefix| never swamps |span sum|
// (SURVEY §7 hard part 2).
//   out_i = C_i/delta_i^{d+2} (h^d c_0 S_i - |B_delta| u_i)        (Mass)
//   out_i = C_i/delta_i^{d+2}  h^d c_0 (S_i - count_i u_i)         (Difference)
#include <algorithm>
#include <vector>

#include <cstdlib>
#include <type_traits>

#include "plan.hpp"

namespace nlg {

namespace {

constexpr int kSeg = 1024;   // scan segment (nodes)
constexpr int kScanThreads = 256;

// Row layout: the scan axis is the fastest one (axis dim-1). For dim = 1 the
// single "row" is the input slab; otherwise rows have length n.
struct RowGeom {
  int64_t rows, len, nseg;
};

// Single-pass row prefix sums with decoupled look-back (one launch, no
// serial offset pass). Tiles of kSeg nodes; a CTA takes the next tile ticket
// (tiles are handed out in row-major order, so every predecessor of a tile is
// already running or done: forward progress without co-residency
// assumptions), scans its tile in double-double, publishes the tile aggregate,
// walks back over its row's predecessors (adding aggregates until it meets an
// inclusive prefix), publishes its own inclusive prefix and writes GLOBAL
// exclusive prefixes P(p) = sum_{q < p} u_q. Flags carry the apply's epoch, so
// nothing is reset between applies.
struct ScanState {
  unsigned long long* ticket;   // tickets handed out (monotone across applies)
  unsigned* flag;               // [tiles] epoch << 2 | {1 aggregate, 2 inclusive}
  double2* agg;                 // [tiles] (hi, lo)
  double2* inc;                 // [tiles] (hi, lo)
};

__device__ __forceinline__ void publish(unsigned* f, unsigned v) {
  __threadfence();
  atomicExch(f, v);
}

__global__ void __launch_bounds__(kScanThreads) scan_lookback(const double* __restrict__ u, RowGeom rg,
                                                             ScanState st, unsigned epoch, unsigned long long base,
                                                             double* __restrict__ pref_hi,
                                                             double* __restrict__ pref_lo,
                                                             double* __restrict__ tot_hi,
                                                             double* __restrict__ tot_lo) {
  constexpr int PER = kSeg / kScanThreads;
  __shared__ unsigned long long s_tile;
  __shared__ double sh[kScanThreads], sl[kScanThreads];
  __shared__ dd s_off;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(st.ticket, 1ull) - base;
  __syncthreads();
  const int64_t tile = static_cast<int64_t>(s_tile);
  const int64_t row = tile / rg.nseg, seg = tile % rg.nseg;
  const int64_t b0 = row * rg.len + seg * kSeg;
  const int64_t lim = min(static_cast<int64_t>(kSeg), rg.len - seg * kSeg);
  double v[PER];
  dd run{0.0, 0.0};
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int64_t p = static_cast<int64_t>(tid) * PER + j;
    v[j] = p < lim ? u[b0 + p] : 0.0;
    run = dd_add(run, {v[j], 0.0});
  }
  // inclusive scan of the thread sums over the CTA: warp shuffles, then the warp totals (three
  // barriers; the shared-memory Hillis-Steele it replaces took sixteen)
  {
    constexpr int NWARP = kScanThreads / 32;
    __shared__ double wh[NWARP], wl[NWARP];
    const int ln = tid & 31, wp = tid >> 5;
    dd inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double hi = __shfl_up_sync(0xffffffffu, inc.hi, o), lo = __shfl_up_sync(0xffffffffu, inc.lo, o);
      if (ln >= o) inc = dd_add(inc, {hi, lo});
    }
    if (ln == 31) {
      wh[wp] = inc.hi;
      wl[wp] = inc.lo;
    }
    __syncthreads();
    if (wp == 0) {
      dd w = ln < NWARP ? dd{wh[ln], wl[ln]} : dd{0.0, 0.0};
#pragma unroll
      for (int o = 1; o < NWARP; o <<= 1) {
        const double hi = __shfl_up_sync(0xffffffffu, w.hi, o), lo = __shfl_up_sync(0xffffffffu, w.lo, o);
        if (ln >= o) w = dd_add(w, {hi, lo});
      }
      if (ln < NWARP) {
        wh[ln] = w.hi;
        wl[ln] = w.lo;
      }
    }
    __syncthreads();
    if (wp > 0) inc = dd_add({wh[wp - 1], wl[wp - 1]}, inc);
    sh[tid] = inc.hi;
    sl[tid] = inc.lo;
    __syncthreads();
  }
  if (tid < 32) {   // warp 0: publish, then look back 32 predecessors at a time
    const int lane = tid;
    const dd agg{sh[kScanThreads - 1], sl[kScanThreads - 1]};
    dd off{0.0, 0.0};
    if (seg == 0) {
      if (lane == 0) {
        st.inc[tile] = make_double2(agg.hi, agg.lo);
        publish(st.flag + tile, epoch << 2 | 2u);
      }
    } else {
      if (lane == 0) {
        st.agg[tile] = make_double2(agg.hi, agg.lo);
        publish(st.flag + tile, epoch << 2 | 1u);
      }
      const int64_t first = tile - seg;                      // first tile of this row
      for (int64_t top = tile - 1;; top -= 32) {
        const int64_t p = top - lane;                        // lane l inspects tile top - l
        const bool valid = p >= first;
        unsigned f = 0;
        if (valid) {
          do {
            f = *reinterpret_cast<volatile unsigned*>(st.flag + p);
          } while ((f >> 2) != epoch);
        }
        __threadfence();
        const unsigned incl = __ballot_sync(0xffffffffu, valid && (f & 3u) == 2u);
        const int stop = incl ? __ffs(incl) - 1 : 32;        // nearest predecessor with an inclusive prefix
        dd v{0.0, 0.0};
        if (valid && lane <= stop) {
          const double2 w = lane == stop ? __ldcg(st.inc + p) : __ldcg(st.agg + p);
          v = {w.x, w.y};
        }
        // warp sum in double-double (fixed tree: deterministic)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const dd u2{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
          v = dd_add(v, u2);
        }
        off = dd_add(off, v);
        if (incl || top - 32 < first) break;
      }
      if (lane == 0) {
        const dd inc = dd_add(off, agg);
        st.inc[tile] = make_double2(inc.hi, inc.lo);
        publish(st.flag + tile, epoch << 2 | 2u);
      }
    }
    if (lane == 0) {
      if (seg == rg.nseg - 1) {
        const dd tot = dd_add(off, agg);
        tot_hi[row] = tot.hi;
        tot_lo[row] = tot.lo;
      }
      s_off = off;
    }
  }
  __syncthreads();
  dd excl = dd_add(s_off, tid ? dd{sh[tid - 1], sl[tid - 1]} : dd{0.0, 0.0});
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int64_t p = static_cast<int64_t>(tid) * PER + j;
    if (p < lim) {
      pref_hi[b0 + p] = excl.hi;
      pref_lo[b0 + p] = excl.lo;
    }
    excl = dd_add(excl, {v[j], 0.0});
  }
}

struct SpanArgs {
  Geom g;
  RowGeom rg;
  const double* u;
  const double* delta;
  double delta0;
  const double* coeff;
  double coeff0;
  double c0;
  int rule, form;
  const double *pref_hi, *pref_lo, *tot_hi, *tot_lo;
  double* out;
  int sym;   // n a power of two: exact coordinates, mirror-symmetric spans
  int intspan;   // span extents from the integer classification (NLG_SPAN_INT=0: predicate probes)
};

// global exclusive prefix P(row, p) for p in [0, len] (P(len) = row total)
__device__ __forceinline__ dd prefix_at(const SpanArgs& a, int64_t row, int64_t p) {
  if (p >= a.rg.len) return {a.tot_hi[row], a.tot_lo[row]};
  return {a.pref_hi[row * a.rg.len + p], a.pref_lo[row * a.rg.len + p]};
}

// Exact membership of source multi-index k for target x (Leaf: cube_intersects_ball
// on the leaf box; Point: dist < delta), same ops as direct.cu.
template <int DIM>
__device__ __forceinline__ bool member(int rule, const int64_t* k, const double* x, double h,
                                       double delta, double r2max) {
  if (rule == 1) {
    double r2 = 0.0;
#pragma unroll
    for (int j = 0; j < DIM; ++j) {
      const double d = __dsub_rn(coord(k[j], h), x[j]);
      r2 = __dadd_rn(r2, __dmul_rn(d, d));
    }
    return __dsqrt_rn(r2) < delta;
  }
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
  return dmin < r2max;
}

// Largest e >= 0 with member(kc + dir*e) along the last axis, given member(kc).
template <int DIM>
__device__ __forceinline__ int64_t span_extent(int rule, int64_t* k, int64_t kc, int dir, const double* x,
                                               double h, double delta, double r2max, int64_t est) {
  int64_t e = est < 0 ? 0 : est;
  k[DIM - 1] = kc + dir * e;
  while (e > 0 && !member<DIM>(rule, k, x, h, delta, r2max)) {
    --e;
    k[DIM - 1] = kc + dir * e;
  }
  for (;;) {
    k[DIM - 1] = kc + dir * (e + 1);
    if (!member<DIM>(rule, k, x, h, delta, r2max)) break;
    ++e;
  }
  return e;
}

// SMALL: (2 delta_max / h)^2 fits 32-bit integers (every 2-D / 3-D horizon of interest): the per-row
// integer classification runs in int instead of int64_t (64-bit multiplies and compares are several
// instructions each; the kernel is issue-bound)
template <int DIM, bool SMALL>
__global__ void __launch_bounds__(256) span_eval(SpanArgs a) {
  using I = typename std::conditional<SMALL, int, int64_t>::type;
  const Geom& g = a.g;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nout = (g.row_end - g.row_begin) * g.stride0;
  // Constant horizon (no delta array): every target shares the row extents, so the CTA tabulates
  // them once per leading offset: entry >= 0 the extent, kExtOut the row is outside, kExtBand a
  // tie band touches the row (the per-target classification below decides).
  constexpr int kExtOut = -1, kExtBand = -2, kTabMax = 441;
  __shared__ int s_ext[kTabMax];
  int tabW = -1;                                        // table half width (leading offsets -W..W), -1: no table
  if (SMALL && DIM > 1 && a.intspan && a.delta == nullptr) {
    const double inv_h0 = 1.0 / g.h, ec = a.delta0 * inv_h0;
    const int W0 = static_cast<int>(floor(a.delta0 / g.h)) + 2, side = 2 * W0 + 1;
    const int cnt = DIM == 2 ? side : side * side;
    if (cnt <= kTabMax) {
      tabW = W0;
      const double E0 = a.rule == 1 ? ec * ec : 4.0 * ec * ec;
      const int lo_ = static_cast<int>(ceil(E0 * (1.0 - tie_band_n(inv_h0))));
      const int hi_ = static_cast<int>(floor(E0 * (1.0 + tie_band_n(inv_h0))));
      auto tm = [&](int d) {
        d = d < 0 ? -d : d;
        const int v = a.rule == 1 ? d : 2 * d - 1;
        return d == 0 ? 0 : v * v;
      };
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        const int d0 = (DIM == 2 ? i : i / side) - W0, d1 = DIM == 2 ? 0 : i % side - W0;
        const int q = tm(d0) + (DIM == 3 ? tm(d1) : 0);
        int e = kExtOut;
        if (q <= hi_) {
          if (q >= lo_) {
            e = kExtBand;
          } else {
            int r = static_cast<int>(sqrtf(static_cast<float>(lo_ - 1 - q)));
            while (r * r > lo_ - 1 - q) --r;
            while ((r + 1) * (r + 1) <= lo_ - 1 - q) ++r;
            e = a.rule == 1 ? r : (r + 1) / 2;
            if (q + tm(e + 1) <= hi_) e = kExtBand;
          }
        }
        s_ext[i] = e;
      }
    }
    __syncthreads();
  }
  if (t >= nout) return;
  int64_t ki[3] = {0, 0, 0};
  {
    int64_t rest = t % g.stride0;
    ki[0] = g.row_begin + t / g.stride0;
    for (int j = DIM - 1; j >= 1; --j) {
      ki[j] = rest % g.n;
      rest /= g.n;
    }
  }
  int64_t ii;
  {
    int64_t rest = 0;
    for (int j = 1; j < DIM; ++j) rest = rest * g.n + ki[j];
    ii = (ki[0] - g.in_begin) * g.stride0 + rest;
  }
  const double h = g.h;
  double x[3];
#pragma unroll
  for (int j = 0; j < DIM; ++j) x[j] = coord(ki[j], h);
  const double delta = a.delta ? a.delta[ii] : a.delta0;
  const double ci = a.coeff ? a.coeff[ii] : a.coeff0;
  const double r2max = __dmul_rn(delta, delta);
  const int64_t W = static_cast<int64_t>(floor(delta / h)) + 2;
  const double rc = delta / h;  // horizon in cells, for span estimates

  dd S{0.0, 0.0};
  int64_t count = 0;
  int64_t k[3] = {0, 0, 0};
  const int64_t lo0 = DIM > 1 ? max(ki[0] - W, int64_t(0)) : 0;
  const int64_t hi0 = DIM > 1 ? min(ki[0] + W, g.n - 1) : 0;
  const int64_t lo1 = DIM > 2 ? max(ki[1] - W, int64_t(0)) : 0;
  const int64_t hi1 = DIM > 2 ? min(ki[1] + W, g.n - 1) : 0;
  // Integer classification of a source at offset d (the stencils' scheme): Point rule |d|^2 against
  // (delta/h)^2; Leaf rule 4 dmin / h^2 = sum_{d_a != 0} (2|d_a| - 1)^2 against (2 delta/h)^2 (the
  // target is a cell centre, the nearest face of cell k lies (|d_a| - 1/2) h away). m < mlo is surely
  // inside, m > mhi surely outside; only inside the tie band does the reference's float predicate
  // decide, so a row's extent is one integer square root instead of a few fp64 predicate probes.
  const double inv_h = 1.0 / h;
  const double ecell = delta * inv_h;
  const double E = a.rule == 1 ? ecell * ecell : 4.0 * ecell * ecell;
  const I mlo = static_cast<I>(ceil(E * (1.0 - tie_band_n(inv_h))));
  const I mhi = static_cast<I>(floor(E * (1.0 + tie_band_n(inv_h))));
  const bool point = a.rule == 1;
  auto term = [&](I d) {   // contribution of one axis offset
    d = d < 0 ? -d : d;
    const I t = point ? d : 2 * d - 1;
    return d == 0 ? I(0) : t * t;
  };
  auto isqrt_i = [](I m) {
    I r = SMALL ? static_cast<I>(sqrtf(static_cast<float>(m))) : static_cast<I>(sqrt(static_cast<double>(m)));
    while (r * r > m) --r;
    while ((r + 1) * (r + 1) <= m) ++r;
    return r;
  };
  for (int64_t a0 = lo0; a0 <= hi0; ++a0) {
    for (int64_t a1 = lo1; a1 <= hi1; ++a1) {
      if (DIM > 1) k[0] = a0;
      if (DIM > 2) k[1] = a1;
      const int64_t kc = ki[DIM - 1];
      k[DIM - 1] = kc;
      int64_t er, el;
      int te = kExtBand;
      if (tabW >= 0) {
        const int side = 2 * tabW + 1;
        const int i0 = static_cast<int>(a0 - ki[0]) + tabW;
        te = s_ext[DIM == 2 ? i0 : i0 * side + static_cast<int>(a1 - ki[1]) + tabW];
        if (te == kExtOut) continue;
      }
      if (te >= 0) {
        er = el = te;
      } else if (a.intspan) {
        I q = 0;
        if (DIM > 1) q += term(static_cast<I>(a0 - ki[0]));
        if (DIM > 2) q += term(static_cast<I>(a1 - ki[1]));
        if (q > mhi) continue;
        if (q >= mlo && !member<DIM>(a.rule, k, x, h, delta, r2max)) continue;
        I ein = 0;                             // largest e with q + term(e) < mlo
        if (q < mlo) {
          const I t = isqrt_i(mlo - 1 - q);
          ein = point ? t : (t + 1) / 2;
        }
        I ir = ein, il = ein;
        if (q + term(ein + 1) <= mhi) {        // tie band: the float predicate, each side on its own
          for (;;) {
            if (q + term(ir + 1) > mhi) break;
            k[DIM - 1] = kc + ir + 1;
            if (!member<DIM>(a.rule, k, x, h, delta, r2max)) break;
            ++ir;
          }
          for (;;) {
            if (q + term(il + 1) > mhi) break;
            k[DIM - 1] = kc - (il + 1);
            if (!member<DIM>(a.rule, k, x, h, delta, r2max)) break;
            ++il;
          }
        }
        er = ir;
        el = il;
      } else {
        if (!member<DIM>(a.rule, k, x, h, delta, r2max)) continue;
        // span estimate from the radius left for this row
        double q = 0.0;
        if (DIM > 1) { const double d = fabs(static_cast<double>(a0 - ki[0])); q += d * d; }
        if (DIM > 2) { const double d = fabs(static_cast<double>(a1 - ki[1])); q += d * d; }
        const int64_t est = static_cast<int64_t>(sqrt(fmax(rc * rc - q, 0.0)));
        er = span_extent<DIM>(a.rule, k, kc, +1, x, h, delta, r2max, est);
        // n = 2^L: node coordinates and cell faces are exact dyadics, so the
        // predicate is mirror-symmetric about the target's cell and the left
        // extent equals the right one (half the probes)
        el = a.sym ? er : span_extent<DIM>(a.rule, k, kc, -1, x, h, delta, r2max, est);
      }
      int64_t lo = kc - el, hi = kc + er;
      lo = max(lo, int64_t(0));
      hi = min(hi, g.n - 1);
      if (lo > hi) continue;
      int64_t row, plo, phi;
      if (DIM == 1) {
        row = 0;
        plo = lo - g.in_begin;
        phi = hi - g.in_begin + 1;
      } else {
        row = (DIM == 2) ? (a0 - g.in_begin) : ((a0 - g.in_begin) * g.n + a1);
        plo = lo;
        phi = hi + 1;
      }
      S = dd_add(S, dd_sub(prefix_at(a, row, phi), prefix_at(a, row, plo)));
      count += hi - lo + 1;
    }
  }
  const double ui = a.u[ii];
  const double front = __ddiv_rn(ci, delta_power(DIM, delta));
  double out;
  if (a.form == 0) {
    out = front * (g.hd * (a.c0 * dd_val(S)) - ball_volume(DIM, delta) * ui);
  } else {
    const dd diff = dd_sub(S, two_sum(static_cast<double>(count) * ui, 0.0));
    out = front * g.hd * (a.c0 * dd_val(diff));
  }
  a.out[t] = out;
}

RowGeom row_geom(const Plan& P) {
  RowGeom rg;
  if (P.geom.dim == 1) {
    rg.rows = 1;
    rg.len = P.n_in;
  } else {
    rg.len = P.geom.n;
    rg.rows = P.n_in / P.geom.n;
  }
  rg.nseg = (rg.len + kSeg - 1) / kSeg;
  return rg;
}

// ---------------------------------------------------------------------------
// 1-D, K >= 1: centred moment scans (the reference's Steps 2 + 3,
// tree.cpp:115-161 and operators.cpp:126-167, re-based). The reference sums
// raw global monomials x^m u and expands (y - x)^{2j} binomially around the
// origin, which loses all digits at small delta (ledger L4).
// Here the moments are centred on short segments: segment s of Ls nodes
// (Ls a power of two <= the smallest horizon in cells) has centre c_s, node k
// the exact half-integer offset t_k = k - c_s, and the scan stores
//   I_m(p) = sum_{k in seg(p), k <= p} t_k^m u_k,   m = 0 .. 2K
// (double-double, inclusive within the segment; no carry between segments:
// the origins differ, and a global carry would bring the conditioning back).
// A target's exact Leaf span [a, b] is cut at segment boundaries; each piece
// contributes its moment differences shifted from c_s to the target by the
// binomial identity (t - d)^{2j} = sum_m C(2j, m) t^m (-d)^{2j-m}, |d| <=
// delta/h + Ls, so the expansion never cancels more than ~4^{2j} ulps:
//   S_i = sum_j c_j (h / delta)^{2j} sum_pieces sum_m C(2j,m) (-d)^{2j-m} dM_m
//   out_i = C_i / delta^3 (h S_i - |B_delta| u_i)                  (Mass form)

constexpr int kMaxMom = 7;   // 2K + 1 for K <= 3

struct MomArgs {
  Geom g;
  int64_t n_in, ls, lshift;   // segment length Ls = 1 << lshift
  int nm, K;
  const double* u;
  const double* delta;
  double delta0;
  const double* coeff;
  double coeff0;
  double c[4];                // p(s) = sum_j c_j s^{2j}
  int rule;
  double* mhi;                // [nm][n_in]
  double* mlo;
  double* out;
};

// one warp per segment, 32-node strides, warp-shuffle inclusive scans in dd
__global__ void __launch_bounds__(256) moment_scan(const __grid_constant__ MomArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t seg = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t s0 = seg << a.lshift;
  if (s0 >= a.n_in) return;
  const double cs = static_cast<double>(a.ls - 1) * 0.5;   // centre (segment-local index)
  dd carry[kMaxMom];
#pragma unroll
  for (int m = 0; m < kMaxMom; ++m) carry[m] = {0.0, 0.0};
  for (int64_t q = 0; q < a.ls; q += 32) {
    const int64_t k = s0 + q + lane;
    const bool in = q + lane < a.ls && k < a.n_in;
    const double uk = in ? a.u[k] : 0.0;
    const double t = static_cast<double>(q + lane) - cs;
    double tm = 1.0;
#pragma unroll
    for (int m = 0; m < kMaxMom; ++m) {
      if (m < a.nm) {
        dd v{tm * uk, fma(tm, uk, -(tm * uk))};        // t^m u as an exact dd product of the double t^m
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double hh = __shfl_up_sync(0xffffffffu, v.hi, o);
          const double ll = __shfl_up_sync(0xffffffffu, v.lo, o);
          if (lane >= o) v = dd_add(v, {hh, ll});
        }
        v = dd_add(v, carry[m]);
        if (in) {
          a.mhi[m * a.n_in + k] = v.hi;
          a.mlo[m * a.n_in + k] = v.lo;
        }
        carry[m] = {__shfl_sync(0xffffffffu, v.hi, 31), __shfl_sync(0xffffffffu, v.lo, 31)};
        tm *= t;
      }
    }
  }
}

__device__ __forceinline__ dd mom_at(const MomArgs& a, int m, int64_t k, int64_t s0) {
  // inclusive in-segment prefix at k, 0 before the segment start
  if (k < s0) return {0.0, 0.0};
  return {a.mhi[m * a.n_in + k], a.mlo[m * a.n_in + k]};
}

__global__ void __launch_bounds__(256) moment_eval(const __grid_constant__ MomArgs a) {
  const Geom& g = a.g;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nout = g.row_end - g.row_begin;
  if (t >= nout) return;
  const int64_t kx = g.row_begin + t;
  const int64_t ii = kx - g.in_begin;
  const double h = g.h;
  double x[1] = {coord(kx, h)};
  const double delta = a.delta ? a.delta[ii] : a.delta0;
  const double ci = a.coeff ? a.coeff[ii] : a.coeff0;
  const double r2max = __dmul_rn(delta, delta);
  const double rc = delta / h;
  int64_t k[1] = {kx};
  double out = 0.0;
  if (member<1>(a.rule, k, x, h, delta, r2max)) {
    const int64_t est = static_cast<int64_t>(rc);
    const int64_t er = span_extent<1>(a.rule, k, kx, +1, x, h, delta, r2max, est);
    const int64_t el = (g.n & (g.n - 1)) == 0 ? er : span_extent<1>(a.rule, k, kx, -1, x, h, delta, r2max, est);
    const int64_t lo = max(kx - el, int64_t(0)) - g.in_begin, hi = min(kx + er, g.n - 1) - g.in_begin;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};   // sum (t - d)^{2j} u over the span, j = 0..K
    for (int64_t s0 = (lo >> a.lshift) << a.lshift; s0 <= hi; s0 += a.ls) {
      const int64_t pa = max(lo, s0), pb = min(hi, s0 + a.ls - 1);
      const double d = static_cast<double>(ii - s0) - static_cast<double>(a.ls - 1) * 0.5;   // target - centre
      double dm[kMaxMom];
#pragma unroll
      for (int m = 0; m < kMaxMom; ++m)
        dm[m] = m < a.nm ? dd_val(dd_sub(mom_at(a, m, pb, s0), mom_at(a, m, pa - 1, s0))) : 0.0;
      // (t - d)^{2j} = sum_m C(2j, m) t^m (-d)^{2j - m}
      double np[kMaxMom];   // (-d)^e
      np[0] = 1.0;
#pragma unroll
      for (int e = 1; e < kMaxMom; ++e) np[e] = np[e - 1] * (-d);
      acc[0] += dm[0];
      if (a.K >= 1) acc[1] += np[2] * dm[0] + 2.0 * np[1] * dm[1] + dm[2];
      if (a.K >= 2) acc[2] += np[4] * dm[0] + 4.0 * np[3] * dm[1] + 6.0 * np[2] * dm[2] + 4.0 * np[1] * dm[3] + dm[4];
      if (a.K >= 3)
        acc[3] += np[6] * dm[0] + 6.0 * np[5] * dm[1] + 15.0 * np[4] * dm[2] + 20.0 * np[3] * dm[3] +
                  15.0 * np[2] * dm[4] + 6.0 * np[1] * dm[5] + dm[6];
    }
    const double q = (h / delta) * (h / delta);   // (h / delta)^2: t is in cells
    double S = 0.0, qj = 1.0;
    for (int j = 0; j <= a.K; ++j) {
      S = fma(a.c[j] * qj, acc[j], S);
      qj *= q;
    }
    const double front = __ddiv_rn(ci, delta_power(1, delta));
    out = front * (g.hd * S - ball_volume(1, delta) * a.u[ii]);
  } else {
    const double front = __ddiv_rn(ci, delta_power(1, delta));
    out = front * (0.0 - ball_volume(1, delta) * a.u[ii]);
  }
  a.out[t] = out;
}

}  // namespace

struct ScanBuffers {
  ScanState st{};
  unsigned epoch = 0;
  unsigned long long tickets = 0;   // handed out so far (host mirror)
  // method 4 (1-D centred moments)
  double* mhi = nullptr;
  double* mlo = nullptr;
  int64_t ls = 0;
  int lshift = 0, K = 0;
};

void spans_setup(Plan& P) {
  const RowGeom rg = row_geom(P);
  P.scan_rows = rg.rows;
  P.scan_len = rg.len;
  P.scan_nseg = rg.nseg;
  const size_t n = static_cast<size_t>(rg.rows * rg.len);
  const size_t tiles = static_cast<size_t>(rg.rows * rg.nseg);
  auto* B = new ScanBuffers();
  P.scan_buf = B;
  NLG_CUDA(cudaMalloc(&P.d_pref_hi, sizeof(double) * n));
  NLG_CUDA(cudaMalloc(&P.d_pref_lo, sizeof(double) * n));
  NLG_CUDA(cudaMalloc(&P.d_seg_hi, sizeof(double) * rg.rows));   // row totals
  NLG_CUDA(cudaMalloc(&P.d_seg_lo, sizeof(double) * rg.rows));
  NLG_CUDA(cudaMalloc(&B->st.ticket, sizeof(unsigned long long)));
  NLG_CUDA(cudaMalloc(&B->st.flag, sizeof(unsigned) * tiles));
  NLG_CUDA(cudaMalloc(&B->st.agg, sizeof(double2) * tiles));
  NLG_CUDA(cudaMalloc(&B->st.inc, sizeof(double2) * tiles));
  NLG_CUDA(cudaMemsetAsync(B->st.ticket, 0, sizeof(unsigned long long), P.stream));
  NLG_CUDA(cudaMemsetAsync(B->st.flag, 0, sizeof(unsigned) * tiles, P.stream));
}

// K >= 1, 1-D: the centred moment scans (fast method 4)
void moments_setup(Plan& P, int K) {
  auto* B = new ScanBuffers();
  P.scan_buf = B;
  B->K = K;
  // segment length: the largest power of two <= the smallest horizon in cells (16 .. 1024)
  double dmin = P.delta0;
  if (P.d_delta) {
    std::vector<double> d(P.n_in);
    NLG_CUDA(cudaMemcpyAsync(d.data(), P.d_delta, sizeof(double) * P.n_in, cudaMemcpyDeviceToHost, P.stream));
    NLG_CUDA(cudaStreamSynchronize(P.stream));
    dmin = *std::min_element(d.begin(), d.end());
  }
  int lsh = 4;
  while (lsh < 10 && static_cast<double>(int64_t{1} << (lsh + 1)) <= dmin / P.geom.h) ++lsh;
  B->lshift = lsh;
  B->ls = int64_t{1} << lsh;
  const size_t nm = static_cast<size_t>(2 * K + 1);
  NLG_CUDA(cudaMalloc(&B->mhi, sizeof(double) * nm * P.n_in));
  NLG_CUDA(cudaMalloc(&B->mlo, sizeof(double) * nm * P.n_in));
  P.fast_method = 4;
}

int64_t moments_segment(const Plan& P) { return P.scan_buf ? P.scan_buf->ls : 0; }

void spans_free(Plan& P) {
  cudaFree(P.d_pref_hi);
  cudaFree(P.d_pref_lo);
  cudaFree(P.d_seg_hi);
  cudaFree(P.d_seg_lo);
  P.d_pref_hi = P.d_pref_lo = P.d_seg_hi = P.d_seg_lo = nullptr;
  if (ScanBuffers* B = P.scan_buf) {
    for (void* p : {static_cast<void*>(B->st.ticket), static_cast<void*>(B->st.flag), static_cast<void*>(B->st.agg),
                    static_cast<void*>(B->st.inc), static_cast<void*>(B->mhi), static_cast<void*>(B->mlo)})
      cudaFree(p);
    delete B;
    P.scan_buf = nullptr;
  }
}

void spans_apply(Plan& P, const double* u, double* out, cudaStream_t s) {
  const RowGeom rg = row_geom(P);
  ScanBuffers& B = *P.scan_buf;
  const unsigned long long tiles = static_cast<unsigned long long>(rg.rows * rg.nseg);
  ++B.epoch;
  if (B.epoch >= (1u << 30)) {   // flag epochs wrap: reset once in a long while
    NLG_CUDA(cudaMemsetAsync(B.st.flag, 0, sizeof(unsigned) * tiles, s));
    B.epoch = 1;
  }
  cudaEvent_t ev;
  stage_begin(P, s, kStSpanScan, &ev);
  scan_lookback<<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(u, rg, B.st, B.epoch, B.tickets, P.d_pref_hi,
                                                                        P.d_pref_lo, P.d_seg_hi, P.d_seg_lo);
  B.tickets += tiles;
  stage_end(P, s, kStSpanScan, ev, 1);
  stage_begin(P, s, kStSpanEval, &ev);
  SpanArgs a;
  a.g = P.geom;
  a.rg = rg;
  a.u = u;
  a.delta = P.d_delta;
  a.delta0 = P.delta0;
  a.coeff = P.d_coeff;
  a.coeff0 = P.coeff0;
  a.c0 = P.prof.poly[0];
  a.rule = P.rule;
  a.form = P.form;
  a.pref_hi = P.d_pref_hi;
  a.pref_lo = P.d_pref_lo;
  a.tot_hi = P.d_seg_hi;
  a.tot_lo = P.d_seg_lo;
  a.out = out;
  a.sym = (P.geom.n & (P.geom.n - 1)) == 0;
  static const bool intspan = [] { const char* e = std::getenv("NLG_SPAN_INT"); return !(e && std::atoi(e) == 0); }();
  a.intspan = intspan;
  const unsigned blocks = static_cast<unsigned>((P.n_out + 255) / 256);
  const double ec = 2.0 * P.delta_max / P.geom.h + 4.0;
  const bool small = ec * ec * P.geom.dim < 1.0e9;      // every integer of the classification below 2^30
  switch (P.geom.dim) {
    case 1: if (small) span_eval<1, true><<<blocks, 256, 0, s>>>(a); else span_eval<1, false><<<blocks, 256, 0, s>>>(a); break;
    case 2: if (small) span_eval<2, true><<<blocks, 256, 0, s>>>(a); else span_eval<2, false><<<blocks, 256, 0, s>>>(a); break;
    default: if (small) span_eval<3, true><<<blocks, 256, 0, s>>>(a); else span_eval<3, false><<<blocks, 256, 0, s>>>(a); break;
  }
  stage_end(P, s, kStSpanEval, ev, 1);
}

void moments_apply(Plan& P, const double* u, double* out, cudaStream_t s) {
  ScanBuffers& B = *P.scan_buf;
  MomArgs a;
  a.g = P.geom;
  a.n_in = P.n_in;
  a.ls = B.ls;
  a.lshift = B.lshift;
  a.K = B.K;
  a.nm = 2 * B.K + 1;
  a.u = u;
  a.delta = P.d_delta;
  a.delta0 = P.delta0;
  a.coeff = P.d_coeff;
  a.coeff0 = P.coeff0;
  for (int j = 0; j < 4; ++j) a.c[j] = j < P.prof.npoly ? P.prof.poly[j] : 0.0;
  a.rule = P.rule;
  a.mhi = B.mhi;
  a.mlo = B.mlo;
  a.out = out;
  cudaEvent_t ev;
  stage_begin(P, s, kStSpanScan, &ev);
  const int64_t nseg = (P.n_in + B.ls - 1) / B.ls;
  moment_scan<<<static_cast<unsigned>((nseg * 32 + 255) / 256), 256, 0, s>>>(a);
  stage_end(P, s, kStSpanScan, ev, 1);
  stage_begin(P, s, kStSpanEval, &ev);
  moment_eval<<<static_cast<unsigned>((P.n_out + 255) / 256), 256, 0, s>>>(a);
  stage_end(P, s, kStSpanEval, ev, 1);
}

}  // namespace nlg
