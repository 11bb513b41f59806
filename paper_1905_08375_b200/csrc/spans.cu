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

// Block-wide exclusive scan of (hi, lo) pairs, kScanThreads threads, each
// owning kSeg / kScanThreads consecutive elements.
__global__ void __launch_bounds__(kScanThreads) scan_segments(const double* __restrict__ u, RowGeom rg,
                                                             double* __restrict__ pref_hi,
                                                             double* __restrict__ pref_lo,
                                                             double* __restrict__ seg_hi,
                                                             double* __restrict__ seg_lo) {
  constexpr int PER = kSeg / kScanThreads;
  const int64_t row = blockIdx.x / rg.nseg;
  const int64_t seg = blockIdx.x % rg.nseg;
  const int64_t base = row * rg.len + seg * kSeg;
  const int64_t lim = min(static_cast<int64_t>(kSeg), rg.len - seg * kSeg);
  const int tid = threadIdx.x;
  double v[PER];
  dd run{0.0, 0.0};
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int64_t p = static_cast<int64_t>(tid) * PER + j;
    v[j] = p < lim ? u[base + p] : 0.0;
    run = dd_add(run, {v[j], 0.0});
  }
  // block scan of per-thread totals (double-double) through shared memory
  __shared__ double sh[kScanThreads], sl[kScanThreads];
  sh[tid] = run.hi;
  sl[tid] = run.lo;
  __syncthreads();
  for (int off = 1; off < kScanThreads; off <<= 1) {
    dd add{0.0, 0.0};
    if (tid >= off) add = {sh[tid - off], sl[tid - off]};
    __syncthreads();
    if (tid >= off) {
      dd cur = dd_add({sh[tid], sl[tid]}, add);
      sh[tid] = cur.hi;
      sl[tid] = cur.lo;
    }
    __syncthreads();
  }
  dd excl = tid ? dd{sh[tid - 1], sl[tid - 1]} : dd{0.0, 0.0};
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int64_t p = static_cast<int64_t>(tid) * PER + j;
    if (p < lim) {
      pref_hi[base + p] = excl.hi;
      pref_lo[base + p] = excl.lo;
    }
    excl = dd_add(excl, {v[j], 0.0});
  }
  if (tid == kScanThreads - 1) {
    seg_hi[row * (rg.nseg + 1) + seg] = sh[tid];
    seg_lo[row * (rg.nseg + 1) + seg] = sl[tid];
  }
}

// Per row: exclusive scan of the segment totals; entry nseg = row total.
__global__ void scan_offsets(RowGeom rg, double* __restrict__ seg_hi, double* __restrict__ seg_lo) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= rg.rows) return;
  double* sh = seg_hi + row * (rg.nseg + 1);
  double* sl = seg_lo + row * (rg.nseg + 1);
  dd run{0.0, 0.0};
  for (int64_t s = 0; s < rg.nseg; ++s) {
    const dd t{sh[s], sl[s]};
    sh[s] = run.hi;
    sl[s] = run.lo;
    run = dd_add(run, t);
  }
  sh[rg.nseg] = run.hi;
  sl[rg.nseg] = run.lo;
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
  const double *pref_hi, *pref_lo, *seg_hi, *seg_lo;
  double* out;
};

// prefix P(row, p) for p in [0, len]
__device__ __forceinline__ dd prefix_at(const SpanArgs& a, int64_t row, int64_t p) {
  const int64_t segs = a.rg.nseg + 1;
  if (p >= a.rg.len) return {a.seg_hi[row * segs + a.rg.nseg], a.seg_lo[row * segs + a.rg.nseg]};
  const int64_t s = p / kSeg;
  const dd off{a.seg_hi[row * segs + s], a.seg_lo[row * segs + s]};
  const dd loc{a.pref_hi[row * a.rg.len + p], a.pref_lo[row * a.rg.len + p]};
  return dd_add(off, loc);
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

template <int DIM>
__global__ void __launch_bounds__(256) span_eval(SpanArgs a) {
  const Geom& g = a.g;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nout = (g.row_end - g.row_begin) * g.stride0;
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
  for (int64_t a0 = lo0; a0 <= hi0; ++a0) {
    for (int64_t a1 = lo1; a1 <= hi1; ++a1) {
      if (DIM > 1) k[0] = a0;
      if (DIM > 2) k[1] = a1;
      const int64_t kc = ki[DIM - 1];
      k[DIM - 1] = kc;
      if (!member<DIM>(a.rule, k, x, h, delta, r2max)) continue;
      // span estimate from the radius left for this row
      double q = 0.0;
      if (DIM > 1) { const double d = fabs(static_cast<double>(a0 - ki[0])); q += d * d; }
      if (DIM > 2) { const double d = fabs(static_cast<double>(a1 - ki[1])); q += d * d; }
      const int64_t est = static_cast<int64_t>(sqrt(fmax(rc * rc - q, 0.0)));
      const int64_t er = span_extent<DIM>(a.rule, k, kc, +1, x, h, delta, r2max, est);
      const int64_t el = span_extent<DIM>(a.rule, k, kc, -1, x, h, delta, r2max, est);
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

}  // namespace

void spans_setup(Plan& P) {
  const RowGeom rg = row_geom(P);
  P.scan_rows = rg.rows;
  P.scan_len = rg.len;
  P.scan_nseg = rg.nseg;
  const size_t n = static_cast<size_t>(rg.rows * rg.len);
  const size_t ns = static_cast<size_t>(rg.rows * (rg.nseg + 1));
  NLG_CUDA(cudaMalloc(&P.d_pref_hi, sizeof(double) * n));
  NLG_CUDA(cudaMalloc(&P.d_pref_lo, sizeof(double) * n));
  NLG_CUDA(cudaMalloc(&P.d_seg_hi, sizeof(double) * ns));
  NLG_CUDA(cudaMalloc(&P.d_seg_lo, sizeof(double) * ns));
}

void spans_free(Plan& P) {
  cudaFree(P.d_pref_hi);
  cudaFree(P.d_pref_lo);
  cudaFree(P.d_seg_hi);
  cudaFree(P.d_seg_lo);
  P.d_pref_hi = P.d_pref_lo = P.d_seg_hi = P.d_seg_lo = nullptr;
}

void spans_apply(Plan& P, const double* u, double* out, cudaStream_t s) {
  const RowGeom rg = row_geom(P);
  const unsigned nblk = static_cast<unsigned>(rg.rows * rg.nseg);
  cudaEvent_t ev;
  stage_begin(P, s, kStSpanScan, &ev);
  scan_segments<<<nblk, kScanThreads, 0, s>>>(u, rg, P.d_pref_hi, P.d_pref_lo, P.d_seg_hi, P.d_seg_lo);
  scan_offsets<<<static_cast<unsigned>((rg.rows + 127) / 128), 128, 0, s>>>(rg, P.d_seg_hi, P.d_seg_lo);
  stage_end(P, s, kStSpanScan, ev, 2);
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
  a.seg_hi = P.d_seg_hi;
  a.seg_lo = P.d_seg_lo;
  a.out = out;
  const unsigned blocks = static_cast<unsigned>((P.n_out + 255) / 256);
  switch (P.geom.dim) {
    case 1: span_eval<1><<<blocks, 256, 0, s>>>(a); break;
    case 2: span_eval<2><<<blocks, 256, 0, s>>>(a); break;
    default: span_eval<3><<<blocks, 256, 0, s>>>(a); break;
  }
  stage_end(P, s, kStSpanEval, ev, 1);
}

}  // namespace nlg
