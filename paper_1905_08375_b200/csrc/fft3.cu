// paper_1905_08375_b200/csrc/fft3.cu — box FFT mode of fast method 3: the
// 3-D fractional operator with a CONSTANT horizon (BASELINE cfg4-A, 768^3,
// delta = 6h) as one fp64 FFT convolution plus an exact tie-band pass.
//
// With a constant horizon every interior target sees the same offset set
// N = {d : |d|^2 < m_lo} (|d|^2 in cells, m_lo the bottom of the tie band
// (delta/h)^2 (1 -+ tie_band), stencil.cu Ball::init), and
//   A_i = sum_{d in N} w(d) u_{i+d},   B_i = sum_{d in N} w(d) (kappa u)_{i+d}
// is a convolution of f = u + i kappa u (two real fields in one complex
// signal) with the real, even kernel w(d) = |d|^-alpha. On a box zero-padded
// in x and y (L >= n + r_f, 2^a 3^b 5^c) it runs in five HBM passes; the x / y
// transforms are Stockham FFTs in shared memory (stockham.cuh), the z
// direction a short direct convolution on the partial spectra:
//   PA  f3_rows<fwd>  : rows (z, y): load u, kappa (the packing), FFT_x -> Z
//   PB  f3_cols       : columns along y (4 kx per CTA): FFT_y
//   PC  f3_zstencil   : per (ky, kx) column the (2 r_f + 1)-tap convolution along
//                       z with G(|dz|; ky, kx) (plan-time partial spectra),
//                       conjugated, in place
//   PD  f3_cols       : FFT_y, only y < n stored
//   PE  f3_rows<inv>  : FFT_x, conjugate: (A, B) of the row, then the combine
//                       out = s (kappa A + B - u diag) of stencil.cu with the
//                       plan's diag / scale (MODE 1 of the stencil: exact sets),
//                       or (A, B) back into the row when the tie pass combines
// conj(F(conj(X))) = L IFFT(X), so the 1 / (L_x L_y) scale is folded into G.
// Offsets in the tie band (|d|^2 in [m_lo, m_hi], e.g. the 30 offsets of
// |d|^2 = 36 at delta = 6h) belong to N_i only where the reference's float
// predicate sqrt(sum (y_j - x_j)^2) < delta on the node coordinates holds
// (operators.cpp:71-78), which varies with the target; f3_ties adds them per
// target with that predicate, so the inclusion set stays bit-exact.
// Sources outside the domain contribute u = 0 (clip and zero collar alike; the
// collar's exterior nodes live in diag), which the zero padding reproduces.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "plan.hpp"
#include "stockham.cuh"

namespace nlg {

constexpr int kTieTX = 32, kTieTY = 8, kTieZC = 128, kMaxTie = 64, kMaxTieR = 16;

struct TieGroups {
  int R, q, ngroup, ntie;   // q: gcd of the t0's (planes z + t0 share z's class mod q)
  int t0[2 * kMaxTieR + 1];
  int beg[2 * kMaxTieR + 2];
  int t1[kMaxTie], t2[kMaxTie];   // ties in t0 order; bit k = k-th tie
  int off[kMaxTie];               // t1 W + t2: offset in the staged window (f3_ties)
};

struct BoxFft {
  int lx = 0, ly = 0, rf = 0;
  int cols = 4;                                     // columns per CTA of the strided passes (NLG_F3_COLS)
  bool tma = false;                                 // PB / PD through bulk tensor copies (NLG_F3_TMA)
  int tma_br = 0;                                   // rows per tensor box
  bool pers = false;                                // PB / PD persistent double-buffered TMA passes (NLG_F3_PERS)
  int pers_ctas = 2;                                // CTAs per SM of the persistent passes
  CUtensorMap pb_in{}, pb_out{}, pd_in{}, pd_out{};
  int64_t n = 0, n_in = 0, o0 = 0, rows_out = 0;   // z: input planes, first output plane, output planes
  double2* z = nullptr;                             // [n_in][ly][lx]: PA / PB output, PC input
  double2* z2 = nullptr;                            // [n_in][ly][lx]: PC output (output planes), PD / PE / ties
  double2* twx = nullptr;                           // [lx] exp(-2 pi i t / lx)
  double2* twy = nullptr;
  double* g = nullptr;                              // [ly][lx][rf + 1] partial spectra / (lx ly)
  int ntie = 0;                                     // tie-band offsets (all |t|^2 = m)
  TieGroups tg{};                                   // ties grouped by t0 (f3_ties)
  int tie_m = 0;                                    // |t|^2 of the band
  double tie_w = 0.0;                               // w_m
  double tie_thr = 0.0;                             // r2 < thr  <=>  sqrt_rn(r2) < delta
  void* tie_mask = nullptr;                         // [n_out] per-target inclusion bits (uint32 / uint64)
  bool tie_tma = false;                             // fixed-band tie pass with the TMA plane ring (f3_ties_tma)
  CUtensorMap tmu{}, tmk{};                         // u, kappa over the input planes: boxes of one window
  const double* tmu_base = nullptr;                 // the u the map tmu was encoded for
};

namespace {

using namespace stockham;

// Strided passes: C = 4 columns per CTA (64-byte row pieces, two CTAs per SM: 3.6 ms per y pass at
// 768^3 against 5.2 ms for C = 8 with one CTA per SM); NLG_F3_COLS=8 (plan time) selects 8.
#ifndef NLG_F3_ROWS_MINB
#define NLG_F3_ROWS_MINB 1            // row passes: resident CTAs per SM the register budget is capped for
#endif
#ifndef NLG_F3_COLS_MINB
#define NLG_F3_COLS_MINB(C) (8 / (C))   // resident CTAs per SM the register budget is capped for
#endif
constexpr int kF3El = 8;     // elements per thread per stage
constexpr int kF3MaxG = 7;   // kernel support radius r_f <= 6 (partial spectra per column in registers)

// Row passes: L / 5 threads for lengths with radix-5 stages (one radix-5
// butterfly per thread: 800-point PA 3.63 ms against 4.47 ms at L / 8, PE in
// (A, B) mode 2.97 against 3.22 ms), except the inverse pass that applies the
// combine, which is faster at L / 8.
template <int L, bool CMB>
__host__ __device__ constexpr int rows_el() { return !CMB && L % 5 == 0 ? 5 : kF3El; }
template <int L, bool CMB>
__host__ __device__ constexpr int rows_threads() {
  return L / rows_el<L, CMB>() < 32 ? 32 : (L / rows_el<L, CMB>() > 256 ? 256 : L / rows_el<L, CMB>());
}
template <int L, int C>
__host__ __device__ constexpr int cols_threads3() { return L * C / kF3El; }

struct F3Args {
  int64_t n, n_in, o0, rows_out;
  int lx, ly, rf;
  const double2* twx;
  const double2* twy;
  const double* g;
  double2* z;
  double2* z2;           // PC writes here (out of place), PD / PE work in it
  int64_t p0, p1;        // plane range of this launch: input planes (PA, PB), output planes (PC, PD, PE)
  const double* u;       // [n_in rows]
  const double* kappa;   // or null
  const double* scale;   // [n_out], or null: scale0 everywhere (constant coefficient)
  double scale0;
  const double* diag;    // [n_out]
  double* out;           // [n_out]
  int ab;                // PE: store (A, B) into the Z row (the tie pass combines)
};

// PA / PE: one row (plane z, row y) per CTA along the contiguous x axis.
// PA: z in [0, n_in); PE: z in output planes, combine into out (or, with a tie
// band, (A, B) back into the row for the tie pass's combine).
// AB (inverse only): store (A, B) into the row (the tie pass combines);
// otherwise the inverse pass applies the combine (and then runs faster at L / 8).
template <int L, bool INV, bool KW, bool AB = false>
__global__ void __launch_bounds__(rows_threads<L, INV && !AB>(), NLG_F3_ROWS_MINB) f3_rows(const __grid_constant__ F3Args a) {
  constexpr int T = rows_threads<L, INV && !AB>();
  __shared__ double2 sm[L + L / 8];
  const int64_t r = blockIdx.x;                      // row within the launch
  const int64_t zr = a.p0 + r / a.n, y = r % a.n;
  const int tid = threadIdx.x;
  if (!INV) {
    const int64_t src = (zr * a.n + y) * a.n;        // u row
    double2* zrow = a.z + (zr * a.ly + y) * a.lx;
    auto ld = [&](int e, int) {
      if (e >= a.n) return make_double2(0.0, 0.0);
      const double v = __ldg(a.u + src + e);
      return make_double2(v, KW ? v * __ldg(a.kappa + src + e) : 0.0);
    };
    auto st = [&](int base, int stride, int, auto& v) {
      constexpr int R = sizeof(v) / sizeof(v[0]);
#pragma unroll
      for (int q = 0; q < R; ++q) zrow[base + q * stride] = v[q];
    };
    fs_fft<false, L, 1, L, 1, T, true>(sm, a.twx, tid, ld, st);
  } else {
    const int64_t zi = a.o0 + zr;                    // input plane of this output plane
    double2* zrow = a.z2 + (zi * a.ly + y) * a.lx;
    const int64_t ii = (zi * a.n + y) * a.n;         // input index of x = 0
    const int64_t oi = (zr * a.n + y) * a.n;         // output index of x = 0
    auto ld = [&](int e, int) { return zrow[e]; };
    auto st = [&](int base, int stride, int, auto& v) {
      constexpr int R = sizeof(v) / sizeof(v[0]);
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int x = base + q * stride;
        if (x < a.n) {
          const double A = v[q].x, B = -v[q].y;      // conjugate: (conv u, conv kappa u)
          if (AB) {                                  // the row's own elements: read before (first stage)
            zrow[x] = make_double2(A, B);
            continue;
          }
          const double X = KW ? fma(__ldg(a.kappa + ii + x), A, B) : A;
          const double sc = a.scale ? __ldg(a.scale + oi + x) : a.scale0;
          a.out[oi + x] = sc * (X - __ldg(a.u + ii + x) * __ldg(a.diag + oi + x));
        }
      }
    };
    fs_fft<false, L, 1, L, 1, T, true>(sm, a.twx, tid, ld, st);
  }
}

// PA with several rows per CTA (RPC): the u and kappa rows of row r + 1
// arrive by 1-D bulk copies (cp.async.bulk, one elected thread, mbarrier
// completion) into a second staging buffer while row r is transformed, so the
// global-load latency that stalled the one-row CTAs (ncu: long-scoreboard
// stalls on the u * kappa products, 63% of the samples,
// profiles/r02_cfg4_ncu_full.json) overlaps the shared-memory stages. Same
// arithmetic as f3_rows. Rows are n contiguous doubles (n * 8 a multiple of 16).
#ifndef NLG_PA_RPC
#define NLG_PA_RPC 4
#endif
template <int L, bool KW>
__global__ void __launch_bounds__(rows_threads<L, false>(), 5) f3_rows_fwd_multi(const __grid_constant__ F3Args a,
                                                                              int64_t rows) {
  constexpr int T = rows_threads<L, false>();
  __shared__ double2 sm[L + L / 8];
  extern __shared__ __align__(128) double stg[];               // [2][KW ? 2 : 1][n]
  __shared__ __align__(8) unsigned long long mbar[2];
  const int tid = threadIdx.x;
  const int n = static_cast<int>(a.n);
  const int F = KW ? 2 : 1;
  const unsigned rb = static_cast<unsigned>(n * sizeof(double));
  const unsigned mb0 = static_cast<unsigned>(__cvta_generic_to_shared(mbar));
  const unsigned s0 = static_cast<unsigned>(__cvta_generic_to_shared(stg));
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * NLG_PA_RPC;
  const int64_t r1 = min(r0 + NLG_PA_RPC, rows);
  auto issue = [&](int64_t r, int buf) {
    const int64_t zr = a.p0 + r / a.n, y = r % a.n;
    const int64_t src = (zr * a.n + y) * a.n;
    const unsigned mb = mb0 + 8u * buf, dst = s0 + static_cast<unsigned>(buf * F) * rb;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(rb * F) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(a.u + src), "r"(rb), "r"(mb)
                 : "memory");
    if (KW)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       dst + rb),
                   "l"(a.kappa + src), "r"(rb), "r"(mb)
                   : "memory");
  };
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (r0 < r1) issue(r0, 0);
  }
  __syncthreads();
  int it = 0;
  for (int64_t r = r0; r < r1; ++r, ++it) {
    const int buf = it & 1;
    if (tid == 0 && r + 1 < r1) issue(r + 1, buf ^ 1);          // its buffer was last read by row r - 1 (barrier below)
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(
            mb0 + 8u * buf),
        "r"(static_cast<unsigned>((it >> 1) & 1))
        : "memory");
    const double* su = stg + static_cast<size_t>(buf * F) * n;
    const int64_t zr = a.p0 + r / a.n, y = r % a.n;
    double2* zrow = a.z + (zr * a.ly + y) * a.lx;
    auto ld = [&](int e, int) {
      if (e >= n) return make_double2(0.0, 0.0);
      const double v = su[e];
      return make_double2(v, KW ? v * su[n + e] : 0.0);
    };
    auto st = [&](int base, int stride, int, auto& v) {
      constexpr int R = sizeof(v) / sizeof(v[0]);
#pragma unroll
      for (int q = 0; q < R; ++q) zrow[base + q * stride] = v[q];
    };
    fs_fft<false, L, 1, L, 1, T, true>(sm, a.twx, tid, ld, st);
    __syncthreads();   // this row's staging and FFT buffers are free for the next issue / row
  }
}

// PB / PD: C adjacent kx columns along y in one plane. PB reads y < n
// (zero padding above) and writes every ky; PD reads every ky and writes y < n.
template <int L, bool PD, int C>
__global__ void __launch_bounds__(cols_threads3<L, C>(), NLG_F3_COLS_MINB(C)) f3_cols(const __grid_constant__ F3Args a) {
  constexpr int T = cols_threads3<L, C>();
  extern __shared__ double2 fsm3[];
  const int tid = threadIdx.x;
  const int kx0 = blockIdx.x * C;
  const int64_t zi = PD ? a.o0 + a.p0 + blockIdx.y : a.p0 + blockIdx.y;
  double2* col = (PD ? a.z2 : a.z) + zi * a.ly * a.lx + kx0;
  auto ld = [&](int e, int c) {
    if (!PD && e >= a.n) return make_double2(0.0, 0.0);
    return col[static_cast<int64_t>(e) * a.lx + c];
  };
  auto st = [&](int base, int stride, int c, auto& v) {
    constexpr int R = sizeof(v) / sizeof(v[0]);
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int e = base + q * stride;
      if (!PD || e < a.n) col[static_cast<int64_t>(e) * a.lx + c] = v[q];
    }
  };
  fs_fft<false, L, 1, L, C, T, false>(fsm3, a.twy, tid, ld, st);
}

// PB / PD with TMA: the CTA's 4-column tile (L rows x 64 bytes, row pitch
// L_x x 16 B) arrives by cp.async.bulk.tensor in boxes of br rows (the tensor
// map's row extent clips: rows beyond it are zero-filled on the load and
// dropped on the store), is transformed in place in shared memory, and leaves
// by bulk tensor stores. No per-thread address arithmetic or 16-byte loads.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int L>
__global__ void __launch_bounds__(cols_threads3<L, 4>(), 2)
    f3_cols_tma(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                const __grid_constant__ F3Args a, int br) {
  constexpr int C = 4, T = cols_threads3<L, C>();
  extern __shared__ __align__(128) double2 fsm3[];
  __shared__ __align__(8) unsigned long long mbar;
  const int tid = threadIdx.x;
  const int cx = blockIdx.x * 2 * C;             // first double of the tile in the row
  const int pz = static_cast<int>(a.p0) + blockIdx.y;   // plane of the view
  const unsigned mb = smem_u32(&mbar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                 "r"(static_cast<unsigned>(L * C * sizeof(double2)))
                 : "memory");
    for (int r0 = 0; r0 < L; r0 += br)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              smem_u32(fsm3 + r0 * C)),
          "l"(&tin), "r"(cx), "r"(r0), "r"(pz), "r"(mb)
          : "memory");
  }
  __syncthreads();
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(mb)
      : "memory");
  auto ld = [&](int e, int c) { return fsm3[e * C + c]; };
  auto st = [&](int base, int stride, int c, auto& v) {
    constexpr int R = sizeof(v) / sizeof(v[0]);
#pragma unroll
    for (int q = 0; q < R; ++q) fsm3[(base + q * stride) * C + c] = v[q];
  };
  fs_fft<false, L, 1, L, C, T, false, true>(fsm3, a.twy, tid, ld, st);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy writes -> the bulk store
  __syncthreads();
  if (tid == 0) {
    for (int r0 = 0; r0 < L; r0 += br)
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tout),
                   "r"(cx), "r"(r0), "r"(pz), "r"(smem_u32(fsm3 + r0 * C))
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// PB / PD, persistent and double buffered: a CTA loops over (column group,
// plane) tiles; the NEXT tile's bulk tensor loads are in flight in the second
// shared-memory buffer while the current tile is transformed, and finished
// tiles leave by bulk tensor stores (the buffer is reloaded only after the
// store has read it: cp.async.bulk.wait_group.read). One elected thread issues
// all copies; the transform is the same in-place Stockham FFT as f3_cols_tma.
template <int L>
__global__ void __launch_bounds__(cols_threads3<L, 4>(), 2)
    f3_cols_pers(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                 const __grid_constant__ F3Args a, int br, int planes) {
  constexpr int C = 4, T = cols_threads3<L, C>();
  constexpr unsigned kTile = static_cast<unsigned>(L * C * sizeof(double2));
  extern __shared__ __align__(128) double2 fsm3[];           // [2][L * C]
  __shared__ __align__(8) unsigned long long mbar[2];
  const int tid = threadIdx.x;
  const int ngx = a.lx / C;
  const int ntile = ngx * planes;
  const unsigned mb0 = smem_u32(mbar), s0 = smem_u32(fsm3);
  auto issue_load = [&](int t, int buf) {
    const int cx = (t % ngx) * 2 * C, pz = static_cast<int>(a.p0) + t / ngx;
    const unsigned mb = mb0 + 8u * buf, dst = s0 + kTile * buf;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(kTile) : "memory");
    for (int r0 = 0; r0 < L; r0 += br)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              dst + static_cast<unsigned>(r0 * C * sizeof(double2))),
          "l"(&tin), "r"(cx), "r"(r0), "r"(pz), "r"(mb)
          : "memory");
  };
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (static_cast<int>(blockIdx.x) < ntile) issue_load(blockIdx.x, 0);
  }
  __syncthreads();
  int it = 0;
  for (int t = blockIdx.x; t < ntile; t += gridDim.x, ++it) {
    const int buf = it & 1;
    const int tn = t + gridDim.x;
    if (tid == 0 && tn < ntile) {
      // the other buffer's store (tile it - 1) must have been read out first
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue_load(tn, buf ^ 1);
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(
            mb0 + 8u * buf),
        "r"(static_cast<unsigned>((it >> 1) & 1))
        : "memory");
    double2* tile = fsm3 + buf * L * C;
    auto ld = [&](int e, int c) { return tile[e * C + c]; };
    auto st = [&](int base, int stride, int c, auto& v) {
      constexpr int R = sizeof(v) / sizeof(v[0]);
#pragma unroll
      for (int q = 0; q < R; ++q) tile[(base + q * stride) * C + c] = v[q];
    };
    stockham::fs_fft<false, L, 1, L, C, T, false, true>(tile, a.twy, tid, ld, st);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy writes -> the bulk store
    __syncthreads();
    if (tid == 0) {
      const int cx = (t % ngx) * 2 * C, pz = static_cast<int>(a.p0) + t / ngx;
      for (int r0 = 0; r0 < L; r0 += br)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tout),
                     "r"(cx), "r"(r0), "r"(pz), "r"(s0 + kTile * buf + static_cast<unsigned>(r0 * C * sizeof(double2)))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// PC: the z direction is not transformed. After FFT_x FFT_y the operator is,
// per column (ky, kx), a (2 r_f + 1)-tap convolution along z with the partial
// spectra G(|dz|; ky, kx) = sum_{dy,dx} w(dz,dy,dx) cos(2 pi ky dy/L_y)
// cos(2 pi kx dx/L_x) / (L_x L_y): 2 r_f + 1 FMA pairs per element instead of
// two padded z transforms. Out of place (Z -> Z2) and cut into z chunks: a
// thread owns one column over zc consecutive output planes, so the grid has
// (columns x chunks) threads and every block of 2 r_f + 1 planes issues all its
// loads before the first FMA (the in-place single-walk version kept one load
// in flight per thread: 34 long-scoreboard stalls per issue, 3.7 TB/s). The
// output planes are stored conjugated for the forward-transform inverses.
template <int RW>
__global__ void __launch_bounds__(256, 2) f3_zstencil(const __grid_constant__ F3Args a, int zc) {
  constexpr int kZW = 2 * RW + 1;
  // one thread per (column, component): the real and imaginary parts of a
  // column are adjacent doubles, so a warp still reads 256 contiguous bytes per
  // plane, and the window + the block's prefetch fit in ~60 registers
  const int64_t plane = static_cast<int64_t>(a.ly) * a.lx;
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= 2 * plane) return;
  const int64_t col = e >> 1;
  const double sgn = (e & 1) ? -1.0 : 1.0;       // conjugate on the store
  // output planes [z0, z1) of this thread, input-plane coordinates
  const int64_t z0 = a.o0 + a.p0 + static_cast<int64_t>(blockIdx.y) * zc;
  const int64_t z1 = min(z0 + zc, a.o0 + a.p1);
  if (z0 >= z1) return;
  double gr[RW + 1];
  {
    const double* gp = a.g + col * (RW + 1);
#pragma unroll
    for (int d = 0; d <= RW; ++d) gr[d] = __ldg(gp + d);
  }
  const double* __restrict__ src = reinterpret_cast<const double*>(a.z) + e;
  double* __restrict__ dst = reinterpret_cast<double*>(a.z2) + e;
  const int64_t nz = a.n_in, pl2 = 2 * plane;
  auto ldz = [&](int64_t zz) { return zz >= 0 && zz < nz ? src[zz * pl2] : 0.0; };
  double win[kZW];                               // slot (p - z0 + RW) % kZW holds plane p
#pragma unroll
  for (int j = 0; j < kZW - 1; ++j) win[j] = ldz(z0 - RW + j);
  for (int64_t zb = z0; zb < z1; zb += kZW) {
    double nx[kZW];                              // the block's new planes, all loads in flight at once
    if (zb + kZW <= z1 && zb + kZW - 1 + RW < nz) {   // interior block: one pointer bumped per load
      const double* p = src + (zb + RW) * pl2;
#pragma unroll
      for (int c = 0; c < kZW; ++c, p += pl2) nx[c] = *p;
    } else {
#pragma unroll
      for (int c = 0; c < kZW; ++c) nx[c] = zb + c < z1 ? ldz(zb + c + RW) : 0.0;
    }
#pragma unroll
    for (int c = 0; c < kZW; ++c) {              // output plane z = zb + c; plane z + k in slot (c + RW + k) % kZW
      const int64_t z = zb + c;
      win[(c + kZW - 1) % kZW] = nx[c];
      if (z < z1) {
        double acc = gr[0] * win[(c + RW) % kZW];
#pragma unroll
        for (int k = 1; k <= RW; ++k) acc = fma(gr[k], win[(c + RW + k) % kZW] + win[(c + RW - k + kZW) % kZW], acc);
        dst[z * pl2] = sgn * acc;
      }
    }
  }
}

// output planes [a.p0, a.p1) in z chunks of about 128 planes
void launch_zstencil(const F3Args& a, cudaStream_t s) {
  const int64_t planes = a.p1 - a.p0;
  if (planes <= 0) return;
  const int64_t nch = std::max<int64_t>(1, (planes + 127) / 128);
  const int zc = static_cast<int>((planes + nch - 1) / nch);
  const dim3 g(static_cast<unsigned>((2 * static_cast<int64_t>(a.ly) * a.lx + 255) / 256), static_cast<unsigned>(nch));
  switch (a.rf) {
    case 1: f3_zstencil<1><<<g, 256, 0, s>>>(a, zc); break;
    case 2: f3_zstencil<2><<<g, 256, 0, s>>>(a, zc); break;
    case 3: f3_zstencil<3><<<g, 256, 0, s>>>(a, zc); break;
    case 4: f3_zstencil<4><<<g, 256, 0, s>>>(a, zc); break;
    case 5: f3_zstencil<5><<<g, 256, 0, s>>>(a, zc); break;
    default: f3_zstencil<6><<<g, 256, 0, s>>>(a, zc); break;
  }
}

// Plan-time partial spectra: G[ky][kx][dz] = 1 / (lx ly)
//   sum_{dy, dx >= 0} m(dy) m(dx) w(dz, dy, dx) cos(2 pi ky dy / ly) cos(2 pi kx dx / lx),
// m(0) = 1, m(>0) = 2 (the kernel is even in every component).
__global__ void f3_spectrum(const double* __restrict__ w, int rf, int lx, int ly, const double* __restrict__ cx,
                            const double* __restrict__ cy, double scale, double* __restrict__ g) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= static_cast<int64_t>(lx) * ly) return;
  const int ky = static_cast<int>(q / lx), kx = static_cast<int>(q % lx);
  const int G = rf + 1;
  for (int dz = 0; dz < G; ++dz) {
    double acc = 0.0;
    for (int dy = 0; dy < G; ++dy) {
      double row = 0.0;
      for (int dx = 0; dx < G; ++dx) {
        const double wv = w[(dz * G + dy) * G + dx];
        if (wv != 0.0) row = fma((dx ? 2.0 : 1.0) * wv, cx[(static_cast<int64_t>(kx) * dx) % lx], row);
      }
      acc = fma((dy ? 2.0 : 1.0) * row, cy[(static_cast<int64_t>(ky) * dy) % ly], acc);
    }
    g[q * G + dz] = scale * acc;
  }
}

// Tie band. Every offset t of the band has the same |t|^2 = m, so one weight
// w_m. Whether t belongs to N_i is the reference's float predicate (exactly as
// stencil.cu point_in), decided once at plan time into a per-target bit mask
// (f3_tie_mask, bit k = tie k, sources outside the domain never set).
// f3_ties then adds  out_i += s_i w_m (kappa_i At_i + Bt_i),  At / Bt the sums
// of u / kappa u over the set bits, sliding along z: a CTA owns a 32 x 8
// column of targets over a chunk of planes of one residue class mod q (q =
// gcd of the tie t0's, 2 at delta = 6h: the sources of plane z are the planes
// z + t0 of the same class). The source planes z - R .. z + R of the class sit
// in a shared-memory ring of NS = 2R/q + 1 staged windows (with an R-cell
// halo, as (u, kappa u) pairs; slot HH W of each reads as zero); each step
// stages ONE new plane, so the L2 traffic per target is ~ (8 + 2R)(32 + 2R) /
// 256 staged pairs instead of one per (target, tie). An excluded tie reads the
// zero slot: no select on the sums.
struct TieArgs {
  Geom g;
  TieGroups tg;
  double w;              // w_m
  double thr;            // r2 < thr  <=>  sqrt_rn(r2) < delta
  const void* mask;      // [n_out] uint32 / uint64
  const double* u;
  const double* kappa;
  const double* scale;   // or null: scale0
  double scale0;
  double* out;
  const double2* zab;    // (A, B) of the FFT convolution in the Z rows: [in plane][y][x], strides below
  int64_t zly, zlx;
  const double* diag;    // [n_out]
  int64_t zlo, zhi;      // target planes [zlo, zhi) of this launch (absolute rows)
};

template <typename MT>
__global__ void f3_tie_mask(const __grid_constant__ TieArgs a, MT* __restrict__ mask) {
  const Geom& g = a.g;
  const int64_t n = g.n;
  const int64_t x = static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x;
  const int64_t y = static_cast<int64_t>(blockIdx.y) * 8 + threadIdx.y;
  const int64_t z = g.row_begin + blockIdx.z;
  if (x >= n || y >= n) return;
  const double h = g.h;
  const double cz = coord(z, h), cy = coord(y, h), cx = coord(x, h);
  MT m = 0;
  for (int gi = 0; gi < a.tg.ngroup; ++gi) {
    const int64_t sz = z + a.tg.t0[gi];
    if (sz < 0 || sz >= n) continue;
    const double d0 = __dsub_rn(coord(sz, h), cz);
    for (int k = a.tg.beg[gi]; k < a.tg.beg[gi + 1]; ++k) {
      const int64_t sy = y + a.tg.t1[k], sx = x + a.tg.t2[k];
      if (sy < 0 || sy >= n || sx < 0 || sx >= n) continue;
      const double d1 = __dsub_rn(coord(sy, h), cy), d2 = __dsub_rn(coord(sx, h), cx);
      const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
      if (r2 < a.thr) m |= static_cast<MT>(1) << k;
    }
  }
  mask[((z - g.row_begin) * n + y) * n + x] = m;
}

constexpr int kTieStage = 4;   // staged (u, kappa) pairs per thread per plane: (8 + 2R)(32 + 2R) <= 1024

// Compile-time tie set of |t|^2 = M, in the host's order (dz, dy, dx ascending).
struct TieSet {
  int n = 0, R = 0, q = 0;
  int t0[kMaxTie] = {}, t1[kMaxTie] = {}, t2[kMaxTie] = {};
  int bit[kMaxTie] = {};   // mask bit: position in the full band's enumeration
};
// DENSE: only the ties without a component of size floor(sqrt(M)) (at M = 36
// the 24 of the (4,4,2) family: R = 4; the 6 axis ties (6,0,0) enter ~2% of
// the targets and are read from global memory in the same pass)
__host__ __device__ constexpr TieSet make_ties(int M, bool dense = false) {
  TieSet s{};
  int Rf = 0;
  while ((Rf + 1) * (Rf + 1) <= M) ++Rf;
  int k = 0;
  for (int dz = -Rf; dz <= Rf; ++dz)
    for (int dy = -Rf; dy <= Rf; ++dy)
      for (int dx = -Rf; dx <= Rf; ++dx)
        if (dz * dz + dy * dy + dx * dx == M) {
          const int az = dz < 0 ? -dz : dz, ay = dy < 0 ? -dy : dy, ax = dx < 0 ? -dx : dx;
          const int mc = az > ay ? (az > ax ? az : ax) : (ay > ax ? ay : ax);
          if ((!dense || mc < Rf) && s.n < kMaxTie) {
            s.t0[s.n] = dz;
            s.t1[s.n] = dy;
            s.t2[s.n] = dx;
            s.bit[s.n] = k;
            s.R = mc > s.R ? mc : s.R;
            ++s.n;
          }
          ++k;
        }
  for (int j = 0; j < s.n; ++j) {   // gcd of the t0's
    int a = s.t0[j] < 0 ? -s.t0[j] : s.t0[j], b = s.q;
    while (b) { const int t = a % b; a = b; b = t; }
    s.q = a;
  }
  if (s.q == 0) s.q = 1;
  return s;
}
// the complement: the axis ties (+-R, 0, 0) and permutations of a band with
// M = R^2 (each enters ~2% of the targets at delta = 6h, 768^3)
__host__ __device__ constexpr TieSet make_axis_ties(int M) {
  TieSet s{};
  int Rf = 0;
  while ((Rf + 1) * (Rf + 1) <= M) ++Rf;
  int k = 0;
  for (int dz = -Rf; dz <= Rf; ++dz)
    for (int dy = -Rf; dy <= Rf; ++dy)
      for (int dx = -Rf; dx <= Rf; ++dx)
        if (dz * dz + dy * dy + dx * dx == M) {
          const int az = dz < 0 ? -dz : dz, ay = dy < 0 ? -dy : dy, ax = dx < 0 ? -dx : dx;
          const int mc = az > ay ? (az > ax ? az : ax) : (ay > ax ? ay : ax);
          if (mc == Rf && s.n < kMaxTie) {
            s.t0[s.n] = dz;
            s.t1[s.n] = dy;
            s.t2[s.n] = dx;
            s.bit[s.n] = k;
            s.R = Rf;
            ++s.n;
          }
          ++k;
        }
  s.q = 1;
  return s;
}
constexpr int kTieFixedM = 36;   // the BASELINE cfg4-A band (delta = 6h): specialised, fully unrolled

// M > 0: the tie set of |t|^2 = M at compile time (offsets, slots and mask
// bits are immediates); M = 0: the runtime set in a.tg.

// build-time experiment knobs (tools/macro_ab.sh): minimum resident CTAs for
// the register budget, the warp-level skip of ties no lane includes, and a
// timing-only variant without the tie sums (wrong results: floor measurement)
#ifndef NLG_TIES_MINB
#define NLG_TIES_MINB 1
#endif
#ifndef NLG_TIES_SKIP
#define NLG_TIES_SKIP 1
#endif
#ifndef NLG_TIES_NOSUM
#define NLG_TIES_NOSUM 0
#endif

template <int M, bool KW, typename MT>
__global__ void __launch_bounds__(kTieTX * kTieTY, NLG_TIES_MINB) f3_ties(const __grid_constant__ TieArgs a) {
  extern __shared__ __align__(16) double2 tsm[];
  const Geom& g = a.g;
  const int n = static_cast<int>(g.n);
  const int64_t nn = g.n * g.n;
  constexpr TieSet TS = make_ties(M, true);           // fixed M: the dense part of the band
  const int R = M ? TS.R : a.tg.R, q = M ? TS.q : a.tg.q, NS = 2 * R / q + 1, NR = NS + 1;
  const int W = kTieTX + 2 * R, SB = (kTieTY + 2 * R) * W, SL = SB + 1;   // slot stride; [SB] = 0
  constexpr int NT = kTieTX * kTieTY;
  const int tid = threadIdx.y * kTieTX + threadIdx.x;
  const int x0 = blockIdx.x * kTieTX, y0 = blockIdx.y * kTieTY;
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  const bool live = x < n && y < n;
  const int cls = static_cast<int>(blockIdx.z) % q;
  const int zb = static_cast<int>(a.zlo) + static_cast<int>(blockIdx.z / q) * kTieZC;
  const int ze = min(static_cast<int>(a.zhi), zb + kTieZC);
  const int zf = zb + ((cls - zb) % q + q) % q;           // first target plane of the class
  if (zf >= ze) return;
  const MT* mask = static_cast<const MT*>(a.mask);
  const int tgt = y * n + x;
  const int sbase = (threadIdx.y + R) * W + threadIdx.x + R;
  for (int sl = tid; sl < NR; sl += NT) tsm[sl * SL + SB] = make_double2(0.0, 0.0);
  if (M > 0)   // the zero block behind the ring (fixed-M excluded ties read it)
    for (int e = tid; e < 2 * (R * W + R) + 8; e += NT) tsm[((NR * SL + 7) & ~7) + e] = make_double2(0.0, 0.0);
  // this thread's staged elements: e = tid + k NT < SB; source offset within a
  // plane (0 outside the domain: the copy then zero-fills)
  int soff[kTieStage];
  unsigned sact = 0, sin_ = 0;
#pragma unroll
  for (int k = 0; k < kTieStage; ++k) {
    const int e = tid + k * NT;
    const int r = e / W, c = e - r * W;
    const int gy = y0 - R + r, gx = x0 - R + c;
    const bool ok = e < SB && gy >= 0 && gy < n && gx >= 0 && gx < n;
    if (e < SB) sact |= 1u << k;
    if (ok) sin_ |= 1u << k;
    soff[k] = ok ? gy * n + gx : 0;
  }
  const unsigned smem0 = static_cast<unsigned>(__cvta_generic_to_shared(tsm)) + 16u * tid;
  // plane p -> slot: (u, kappa) pairs by cp.async, zero outside the domain;
  // the plane base pointers once per plane, per element one add and the copy
  auto stage = [&](int p, int slot) {
    const bool pin = p >= 0 && p < n;
    const int64_t pb = (static_cast<int64_t>(pin ? p : g.in_begin) - g.in_begin) * nn;
    const double* ub = a.u + pb;
    const double* kb = KW ? a.kappa + pb : nullptr;
    const unsigned d0 = smem0 + 16u * static_cast<unsigned>(slot * SL);
#pragma unroll
    for (int k = 0; k < kTieStage; ++k) {
      if (sact & (1u << k)) {
        const unsigned sz = pin && (sin_ & (1u << k)) ? 8u : 0u;
        const unsigned d = d0 + 16u * k * NT;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(ub + soff[k]), "r"(sz) : "memory");
        if (KW)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d + 8u), "l"(kb + soff[k]), "r"(sz)
                       : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // ring of NR = NS + 1 slots: plane zf - R + i q in slot i mod NR
  for (int i = 0; i < NS; ++i) stage(zf - R + i * q, i);
  // per-target operands of plane z, fetched one step ahead: the mask, the
  // FFT's (A, B), diag, scale (the target's own u, kappa are in the ring)
  MT m = 0, mn = 0;
  double2 ab = make_double2(0.0, 0.0), abn = ab;
  double ed = 0.0, es = 0.0, edn = 0.0, esn = 0.0;
  auto fetch = [&](int z) {
    mn = 0;
    abn = make_double2(0.0, 0.0);
    edn = esn = 0.0;
    if (live && z < ze) {
      const int64_t oi = (static_cast<int64_t>(z) - g.row_begin) * nn + tgt;
      const int64_t zi = static_cast<int64_t>(z) - g.in_begin;
      mn = __ldg(mask + oi);
      abn = a.zab[(zi * a.zly + y) * a.zlx + x];
      edn = __ldg(a.diag + oi);
      esn = a.scale ? __ldg(a.scale + oi) : a.scale0;
    }
  };
  fetch(zf);
  int head = 0;                                           // slot of plane zt - R
  for (int zt = zf; zt < ze; zt += q) {
    m = mn;
    ab = abn;
    ed = edn;
    es = esn;
    const int64_t oi = (static_cast<int64_t>(zt) - g.row_begin) * nn + tgt;
    asm volatile("cp.async.wait_all;\n" ::: "memory");   // planes zt - R .. zt + R (own copies)
    __syncthreads();                                      // everyone's copies; last step's reads done
    const int sn = head == 0 ? NR - 1 : head - 1;          // slot of plane zt - R - q: free now
    if (zt + q < ze) stage(zt + q + R, sn);               // next step's plane in flight during the sums
    fetch(zt + q);
    double A = 0.0, B = 0.0;
    if constexpr (M > 0) {
      // axis ties (outside the staged window): the few included sources straight
      // from global memory, loads issued before the window sums (predicated per lane)
      constexpr TieSet AX = make_axis_ties(M);
      double xu[AX.n > 0 ? AX.n : 1], xk[AX.n > 0 ? AX.n : 1];
      {
        const int64_t ii = (static_cast<int64_t>(zt) - g.in_begin) * nn + tgt;
#pragma unroll
        for (int k = 0; k < AX.n; ++k) {
          const bool on = (m >> AX.bit[k]) & 1u;
          const int64_t s = ii + (static_cast<int64_t>(AX.t0[k]) * n + AX.t1[k]) * n + AX.t2[k];
          xu[k] = on ? __ldg(a.u + s) : 0.0;
          xk[k] = on && KW ? __ldg(a.kappa + s) : 0.0;
        }
      }
      constexpr int kNS = 2 * TS.R / TS.q + 1;
      const double2* slot[kNS];
#pragma unroll
      for (int r = 0; r < kNS; ++r) slot[r] = tsm + (head + r < NR ? head + r : head + r - NR) * SL + sbase;
      constexpr int kZH = TS.R * (kTieTX + 2 * TS.R) + TS.R;   // largest |tie offset| in a window
      // Excluded ties read a zero block through the same immediate offset (one
      // SEL of the base per tie, no select on the sums). The zero base of slot
      // r is congruent to the slot's own base mod 8 elements (128 B), so a
      // warp mixing real and zero reads still hits each bank once per quarter.
      const int zb0 = (NR * SL + 7) & ~7;                  // 8-aligned zero block, 2 kZH + 8 elements
      const double2* zc[kNS];
#pragma unroll
      for (int r = 0; r < kNS; ++r) {
        const int sr = static_cast<int>(slot[r] - tsm);
        zc[r] = tsm + zb0 + kZH + (((sr - (zb0 + kZH)) % 8) + 8) % 8;
      }
      // ties no lane of the warp includes are skipped (the inclusion pattern is
      // smooth along x: ~15 of the 24 are needed per warp at 768^3)
      const unsigned wm = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(m));
      double A1 = 0.0, B1 = 0.0;                          // two chains per field
#pragma unroll
      for (int k = 0; k < (NLG_TIES_NOSUM ? 0 : TS.n); ++k) {
        if (NLG_TIES_SKIP && !(wm & (1u << TS.bit[k]))) continue;
        const int r = (TS.t0[k] + TS.R) / TS.q;
        const double2* base = (m & (1u << TS.bit[k])) ? slot[r] : zc[r];
        const double2 v = base[TS.t1[k] * (kTieTX + 2 * TS.R) + TS.t2[k]];
        if (k & 1) {
          A1 += v.x;
          if (KW) B1 = fma(v.x, v.y, B1);
        } else {
          A += v.x;
          if (KW) B = fma(v.x, v.y, B);
        }
      }
      A += A1;
      B += B1;
#pragma unroll
      for (int k = 0; k < AX.n; ++k) {
        A += xu[k];
        if (KW) B = fma(xu[k], xk[k], B);
      }
    } else {
      if (m) {
        for (int gi = 0; gi < a.tg.ngroup; ++gi) {
          int sl = head + (a.tg.t0[gi] + R) / q;
          sl = sl >= NR ? sl - NR : sl;
          const double2* st = tsm + sl * SL;
          const int kb = a.tg.beg[gi], kend = a.tg.beg[gi + 1];
#pragma unroll 4
          for (int k = kb; k < kend; ++k) {             // an excluded tie reads the zero slot
            const double2 v = st[(m >> k) & 1 ? sbase + a.tg.off[k] : SB];
            A += v.x;
            if (KW) B = fma(v.x, v.y, B);
          }
        }
      }
    }
    if (live) {   // the combine of stencil.cu: out = s (kappa (A + w At) + B + w Bt - u diag)
      const double2 own = tsm[(head + R / q < NR ? head + R / q : head + R / q - NR) * SL + sbase];
      const double uA = fma(a.w, A, ab.x);
      const double X = KW ? fma(own.y, uA, fma(a.w, B, ab.y)) : uA;
      a.out[oi] = es * (X - own.x * ed);
    }
    head = head + 1 == NR ? 0 : head + 1;
  }
}

// Tie pass, fixed band (|t|^2 = kTieFixedM), fed by TMA. Same sums and
// combine as f3_ties; the source planes of the residue class arrive in a ring
// of NR = NS + 2 slots by cp.async.bulk.tensor (one elected thread, boxes of
// the (8 + 2R) x (32 + 2R) window of u and of kappa, zero fill outside the
// domain by the tensor map's bounds), each slot completing on its own
// mbarrier, two planes ahead of the step that first reads them: the threads
// issue no staging instructions and the plane latency is hidden by two steps
// of sums. Measured on the cp.async version: without its tie sums the pass
// still took 7.1 of 9.9 ms (staging / operand latency, one step ahead).
__device__ __forceinline__ void mbar_wait(unsigned mb, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(mb),
      "r"(parity)
      : "memory");
}

template <bool KW>
__global__ void __launch_bounds__(kTieTX * kTieTY, 3)
    f3_ties_tma(const __grid_constant__ CUtensorMap tmu, const __grid_constant__ CUtensorMap tmk,
                const __grid_constant__ TieArgs a) {
  constexpr TieSet TS = make_ties(kTieFixedM, true);
  constexpr TieSet AX = make_axis_ties(kTieFixedM);
  constexpr int R = TS.R, q = TS.q, NS = 2 * R / q + 1, NR = NS + 2;
  constexpr int W = kTieTX + 2 * R, SB = (kTieTY + 2 * R) * W;      // window elements
  constexpr int SLOT = (KW ? 2 : 1) * SB;                             // doubles per ring slot
  constexpr unsigned BYTES = sizeof(double) * SLOT;
  extern __shared__ __align__(128) double rsm[];
  __shared__ __align__(8) unsigned long long mbar[NR];
  const Geom& g = a.g;
  const int n = static_cast<int>(g.n);
  const int64_t nn = g.n * g.n;
  const int tid = threadIdx.y * kTieTX + threadIdx.x;
  const int x0 = blockIdx.x * kTieTX, y0 = blockIdx.y * kTieTY;
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  const bool live = x < n && y < n;
  const int cls = static_cast<int>(blockIdx.z) % q;
  const int zb = static_cast<int>(a.zlo) + static_cast<int>(blockIdx.z / q) * kTieZC;
  const int ze = min(static_cast<int>(a.zhi), zb + kTieZC);
  const int zf = zb + ((cls - zb) % q + q) % q;                      // first target plane of the class
  if (zf >= ze) return;
  const int J = (ze - zf + q - 1) / q;                                // target planes of this CTA
  const int NP = J + NS - 1;                                          // source planes: zf - R + i q, i < NP
  const unsigned mb0 = static_cast<unsigned>(__cvta_generic_to_shared(mbar));
  const unsigned sm0 = static_cast<unsigned>(__cvta_generic_to_shared(rsm));
  auto issue = [&](int i) {                                           // plane i -> slot i % NR (thread 0)
    const int sl = i % NR;
    const unsigned mb = mb0 + 8u * sl, dst = sm0 + static_cast<unsigned>(sizeof(double)) * SLOT * sl;
    const int pz = zf - R + i * q - static_cast<int>(g.in_begin);      // input plane (out of range: zero fill)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(BYTES) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(&tmu), "r"(x0 - R), "r"(y0 - R), "r"(pz), "r"(mb)
        : "memory");
    if (KW)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              dst + static_cast<unsigned>(sizeof(double)) * SB),
          "l"(&tmk), "r"(x0 - R), "r"(y0 - R), "r"(pz), "r"(mb)
          : "memory");
  };
  if (tid == 0) {
    for (int i = 0; i < NR; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8u * i) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int i = 0; i < min(NS + 1, NP); ++i) issue(i);
  }
  __syncthreads();
  auto wait_plane = [&](int i) { mbar_wait(mb0 + 8u * (i % NR), static_cast<unsigned>((i / NR) & 1)); };
  for (int i = 0; i < NS - 1; ++i) wait_plane(i);
  const int tgt = y * n + x;
  const int sbase = (threadIdx.y + R) * W + threadIdx.x + R;
  // running pointers to the target plane zt's operands (advanced by q planes a
  // step: no per-step 64-bit index arithmetic); dead lanes point at target 0
  const int64_t step_n = static_cast<int64_t>(q) * nn, step_z = static_cast<int64_t>(q) * a.zly * a.zlx;
  const int64_t t0i = live ? tgt : 0;
  const int64_t oi0 = (static_cast<int64_t>(zf) - g.row_begin) * nn + t0i;
  const int64_t ii0 = (static_cast<int64_t>(zf) - g.in_begin) * nn + t0i;
  const uint32_t* pm = static_cast<const uint32_t*>(a.mask) + oi0;
  const double2* pab = a.zab + ((static_cast<int64_t>(zf) - g.in_begin) * a.zly + (live ? y : 0)) * a.zlx + (live ? x : 0);
  const double* pd = a.diag + oi0;
  const double* ps = a.scale ? a.scale + oi0 : nullptr;
  double* po = a.out + oi0;
  const double* pu = a.u + ii0;
  const double* pkp = KW ? a.kappa + ii0 : nullptr;
  int64_t axoff[AX.n > 0 ? AX.n : 1];
#pragma unroll
  for (int k = 0; k < AX.n; ++k) axoff[k] = (static_cast<int64_t>(AX.t0[k]) * n + AX.t1[k]) * n + AX.t2[k];
  uint32_t mn = 0;
  double2 abn = make_double2(0.0, 0.0);
  double edn = 0.0, esn = 0.0;
  if (live) {   // plane zf
    mn = __ldg(pm);
    abn = pab[0];
    edn = __ldg(pd);
    esn = ps ? __ldg(ps) : a.scale0;
  }
  for (int j = 0; j < J; ++j) {
    const int zt = zf + j * q;
    const uint32_t m = mn;
    const double2 ab = abn;
    const double ed = edn, es = esn;
    __syncthreads();                                                  // step j - 1's reads done: slot of plane j - 1 free
    if (tid == 0 && j + NS + 1 < NP) issue(j + NS + 1);               // two planes ahead
    wait_plane(j + NS - 1);                                           // the newest plane this step reads
    const bool more = live && zt + q < ze;
    mn = more ? __ldg(pm + step_n) : 0u;                              // the next step's operands, one step ahead
    abn = more ? pab[step_z] : make_double2(0.0, 0.0);
    edn = more ? __ldg(pd + step_n) : 0.0;
    esn = more ? (ps ? __ldg(ps + step_n) : a.scale0) : 0.0;
    if (live && zt + 2 * q < ze) {                                    // and the one after that into L2
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pab + 2 * step_z));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pd + 2 * step_n));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pm + 2 * step_n));
    }
    // ties no lane of the warp includes are skipped (~15 of 24 ring ties needed
    // per warp at 768^3; the axis ties enter ~2% of the targets)
    const unsigned wm = __reduce_or_sync(0xffffffffu, m);
    // axis ties (outside the window): the few included sources from global memory
    double xu[AX.n > 0 ? AX.n : 1], xk[AX.n > 0 ? AX.n : 1];
#pragma unroll
    for (int k = 0; k < AX.n; ++k) {
      xu[k] = xk[k] = 0.0;
      if (wm & (1u << AX.bit[k])) {
        const bool on = (m >> AX.bit[k]) & 1u;
        xu[k] = on ? __ldg(pu + axoff[k]) : 0.0;
        xk[k] = on && KW ? __ldg(pkp + axoff[k]) : 0.0;
      }
    }
    const double* slot[NS];
#pragma unroll
    for (int r = 0; r < NS; ++r) slot[r] = rsm + ((j + r) % NR) * SLOT + sbase;
    double A = 0.0, B = 0.0, A1 = 0.0, B1 = 0.0;
#pragma unroll
    for (int k = 0; k < TS.n; ++k) {
      if (!(wm & (1u << TS.bit[k]))) continue;
      const double* sp = slot[(TS.t0[k] + R) / q] + TS.t1[k] * W + TS.t2[k];
      const double uu = (m & (1u << TS.bit[k])) ? sp[0] : 0.0;
      if (k & 1) {
        A1 += uu;
        if (KW) B1 = fma(uu, sp[SB], B1);
      } else {
        A += uu;
        if (KW) B = fma(uu, sp[SB], B);
      }
    }
    A += A1;
    B += B1;
#pragma unroll
    for (int k = 0; k < AX.n; ++k) {
      A += xu[k];
      if (KW) B = fma(xu[k], xk[k], B);
    }
    if (live) {   // out = s (kappa (A + w At) + B + w Bt - u diag); own u, kappa from the ring
      const double* own = slot[R / q];
      const double uA = fma(a.w, A, ab.x);
      const double X = KW ? fma(own[SB], uA, fma(a.w, B, ab.y)) : uA;
      *po = es * (X - own[0] * ed);
    }
    pm += step_n;
    pab += step_z;
    pd += step_n;
    if (ps) ps += step_n;
    po += step_n;
    pu += step_n;
    if (KW) pkp += step_n;
  }
}

// supported axis lengths 2^a 3^b 5^c (multiples of 8 columns, <= 1024 threads per column CTA)
#define NLG_F3_L(X) \
  X(48) X(64) X(72) X(80) X(96) X(128) X(144) X(160) X(192) X(256) X(288) X(384) X(400) X(512) X(576) X(768) \
  X(800) X(864) X(1024)

bool f3_supported(int L) {
#define NLG_F3_CASE(N) if (L == N) return true;
  NLG_F3_L(NLG_F3_CASE)
#undef NLG_F3_CASE
  return false;
}

int f3_length(int64_t need) {
  const int c[] = {48, 64, 72, 80, 96, 128, 144, 160, 192, 256, 288, 384, 400, 512, 576, 768, 800, 864, 1024};
  for (int L : c)
    if (L >= need) return L;
  return 0;
}

template <int L, int C>
size_t cols_smem3() { return sizeof(double2) * L * C; }

template <int L, int C>
void f3_attr_c(int rf) {
  NLG_CUDA(cudaFuncSetAttribute(f3_cols<L, false, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(cols_smem3<L, C>())));
  NLG_CUDA(cudaFuncSetAttribute(f3_cols<L, true, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(cols_smem3<L, C>())));
}
template <int L>
void f3_attr(int rf) {
  f3_attr_c<L, 8>(rf);
  f3_attr_c<L, 4>(rf);
  f3_attr_c<L, 2>(rf);
  NLG_CUDA(cudaFuncSetAttribute(f3_cols_pers<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(2 * sizeof(double2) * L * 4)));
  NLG_CUDA(cudaFuncSetAttribute(f3_cols_tma<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(double2) * L * 4)));
}

template <int L>
void launch_rows(const F3Args& a, bool inv, int64_t rows, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(rows);
  constexpr int TF = rows_threads<L, false>(), TI = rows_threads<L, true>();
  if (!inv) {
    // NLG_PA_MULTI=1: bulk-copy-fed multi-row PA (measured 4.5 vs 3.7 ms at 768^3: off)
    static const bool multi = [] { const char* e = std::getenv("NLG_PA_MULTI"); return e && std::atoi(e) == 1; }();
    if (NLG_PA_RPC > 1 && multi && (a.n * 8) % 16 == 0) {
      const unsigned g2 = static_cast<unsigned>((rows + NLG_PA_RPC - 1) / NLG_PA_RPC);
      const size_t sb = sizeof(double) * 2 * (a.kappa ? 2 : 1) * a.n;
      if (a.kappa) f3_rows_fwd_multi<L, true><<<g2, TF, sb, s>>>(a, rows);
      else f3_rows_fwd_multi<L, false><<<g2, TF, sb, s>>>(a, rows);
    } else if (a.kappa) {
      f3_rows<L, false, true><<<grid, TF, 0, s>>>(a);
    } else {
      f3_rows<L, false, false><<<grid, TF, 0, s>>>(a);
    }
  } else if (a.ab) {
    f3_rows<L, true, false, true><<<grid, TF, 0, s>>>(a);
  } else {
    if (a.kappa) f3_rows<L, true, true><<<grid, TI, 0, s>>>(a);
    else f3_rows<L, true, false><<<grid, TI, 0, s>>>(a);
  }
}

template <int L, int C>
void launch_cols_c(const F3Args& a, bool pd, int64_t planes, cudaStream_t s) {
  const dim3 grid(static_cast<unsigned>(a.lx / C), static_cast<unsigned>(planes));
  if (pd) f3_cols<L, true, C><<<grid, cols_threads3<L, C>(), cols_smem3<L, C>(), s>>>(a);
  else f3_cols<L, false, C><<<grid, cols_threads3<L, C>(), cols_smem3<L, C>(), s>>>(a);
}
template <int L>
void launch_cols_pers(const BoxFft& B, const F3Args& a, bool pd, int64_t planes, cudaStream_t s) {
  static int nsm = 0;
  if (!nsm) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t ntile = static_cast<int64_t>(a.lx / 4) * planes;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ntile, static_cast<int64_t>(B.pers_ctas) * nsm));
  const size_t sb = 2 * sizeof(double2) * L * 4;
  if (pd) f3_cols_pers<L><<<grid, cols_threads3<L, 4>(), sb, s>>>(B.pd_in, B.pd_out, a, B.tma_br, static_cast<int>(planes));
  else f3_cols_pers<L><<<grid, cols_threads3<L, 4>(), sb, s>>>(B.pb_in, B.pb_out, a, B.tma_br, static_cast<int>(planes));
}
template <int L>
void launch_cols_tma(const BoxFft& B, const F3Args& a, bool pd, int64_t planes, cudaStream_t s) {
  const dim3 grid(static_cast<unsigned>(a.lx / 4), static_cast<unsigned>(planes));
  const size_t sb = sizeof(double2) * L * 4;
  if (pd) f3_cols_tma<L><<<grid, cols_threads3<L, 4>(), sb, s>>>(B.pd_in, B.pd_out, a, B.tma_br);
  else f3_cols_tma<L><<<grid, cols_threads3<L, 4>(), sb, s>>>(B.pb_in, B.pb_out, a, B.tma_br);
}

template <int L>
void launch_cols(const F3Args& a, int cols, bool pd, int64_t planes, cudaStream_t s) {
  if (cols == 4) launch_cols_c<L, 4>(a, pd, planes, s);
  else if (cols == 2) launch_cols_c<L, 2>(a, pd, planes, s);
  else launch_cols_c<L, 8>(a, pd, planes, s);
}

std::vector<double2> twiddles3(int n) {
  std::vector<double2> t(n);
  const long double pi2 = 2.0L * std::acos(-1.0L);
  for (int i = 0; i < n; ++i) {
    const long double ang = pi2 * static_cast<long double>(i) / static_cast<long double>(n);
    t[i] = make_double2(static_cast<double>(std::cos(ang)), static_cast<double>(-std::sin(ang)));
  }
  return t;
}
std::vector<double> costab(int n) {
  std::vector<double> t(n);
  const long double pi2 = 2.0L * std::acos(-1.0L);
  for (int i = 0; i < n; ++i) t[i] = static_cast<double>(std::cos(pi2 * static_cast<long double>(i) / n));
  return t;
}

F3Args args_of(const Plan& P, const BoxFft& B) {
  F3Args a;
  a.n = B.n;
  a.n_in = B.n_in;
  a.o0 = B.o0;
  a.rows_out = B.rows_out;
  a.lx = B.lx;
  a.ly = B.ly;
  a.rf = B.rf;
  a.twx = B.twx;
  a.twy = B.twy;
  a.g = B.g;
  a.z = B.z;
  a.z2 = B.z2;
  a.p0 = 0;
  a.p1 = 0;
  a.u = nullptr;
  a.kappa = P.d_kappa;
  a.scale = nullptr;
  a.scale0 = 0.0;
  a.diag = nullptr;
  a.out = nullptr;
  a.ab = 0;
  return a;
}

// smallest double x with sqrt_rn(x) >= delta (host; IEEE sqrt is correctly rounded)
double sqrt_threshold_host(double delta) {
  double t = delta * delta;
  while (t > 0.0 && std::sqrt(t) >= delta) t = std::nextafter(t, 0.0);
  while (std::sqrt(t) < delta) t = std::nextafter(t, 1e300);
  return t;
}

TieArgs tie_args(const Plan& P, const BoxFft& B) {
  TieArgs t;
  t.g = P.geom;
  t.tg = B.tg;
  t.w = B.tie_w;
  t.thr = B.tie_thr;
  t.mask = B.tie_mask;
  t.u = nullptr;
  t.kappa = P.d_kappa;
  t.scale = nullptr;
  t.scale0 = 0.0;
  t.out = nullptr;
  t.zab = B.z2;
  t.zly = B.ly;
  t.zlx = B.lx;
  t.diag = nullptr;
  t.zlo = P.geom.row_begin;
  t.zhi = P.geom.row_end;
  return t;
}


// 3-D tensor map over Z viewed as doubles: (2 L_x, rows, planes), row pitch
// L_x complex, plane pitch L_y L_x complex; boxes of (8 doubles, br rows, 1).
bool encode_cols_map(CUtensorMap* m, void* base, int lx, int ly, int64_t rows, int64_t planes, int br) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return false;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(2 * lx), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(planes)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(lx) * 16, static_cast<cuuint64_t>(ly) * lx * 16};
  const cuuint32_t box[3] = {8, static_cast<cuuint32_t>(br), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D tensor map over an input field (x: n, y: n, z: input planes) with
// boxes of one tie window ((32 + 2R) x (8 + 2R) x 1); out-of-bounds boxes
// are zero filled (the domain / slab edges).
bool encode_window_map(CUtensorMap* m, const double* base, int64_t n, int64_t planes, int R) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess || !fn)
      return false;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if ((n * 8) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(planes)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(n) * 8, static_cast<cuuint64_t>(n) * n * 8};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(kTieTX + 2 * R), static_cast<cuuint32_t>(kTieTY + 2 * R), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// Box FFT mode applies to the 3-D fractional operator with a constant horizon
// (no delta array). NLG_BOX_FFT=0 (environment, read at plan time) keeps the
// stencil sweep.
BoxFft* boxfft_setup(const Plan& P, double alpha) {
  const Geom& g = P.geom;
  const char* env = std::getenv("NLG_BOX_FFT");
  if (env && std::atoi(env) == 0) return nullptr;
  if (g.dim != 3 || P.d_delta || P.family != NLG_FRACTIONAL) return nullptr;
  // tie band exactly as stencil.cu Ball::init
  const double e = P.delta0 / g.h, e2 = e * e;
  const int mlo = static_cast<int>(std::ceil(e2 * (1.0 - tie_band(g.h))));
  const int mhi = static_cast<int>(std::floor(e2 * (1.0 + tie_band(g.h))));
  int rf = 0;
  while ((rf + 1) * (rf + 1) < mlo) ++rf;         // largest component inside the strict ball
  if (rf < 1 || rf + 1 > kF3MaxG) return nullptr;
  const int64_t n = g.n, n_in = g.in_end - g.in_begin;
  const int lx = f3_length(n + rf);
  if (!lx || !f3_supported(lx)) return nullptr;
  auto* B = new BoxFft();
  B->lx = B->ly = lx;
  B->rf = rf;
  if (const char* ce = std::getenv("NLG_F3_COLS")) B->cols = std::atoi(ce) == 8 ? 8 : (std::atoi(ce) == 2 ? 2 : 4);
  B->n = n;
  B->n_in = n_in;
  B->o0 = P.halo_lo;
  B->rows_out = g.row_end - g.row_begin;
  const int G = rf + 1;
  std::vector<double> w(static_cast<size_t>(G) * G * G, 0.0);
  for (int dz = 0; dz < G; ++dz)
    for (int dy = 0; dy < G; ++dy)
      for (int dx = 0; dx < G; ++dx) {
        const int m = dz * dz + dy * dy + dx * dx;
        if (m > 0 && m < mlo) w[(dz * G + dy) * G + dx] = std::pow(static_cast<double>(m), -0.5 * alpha);
      }
  // tie band: one |t|^2 = m (the band is narrower than 1), grouped by t0
  if (mlo <= mhi) {
    TieGroups& tg = B->tg;
    const int m = mlo;
    const int R = static_cast<int>(std::floor(std::sqrt(static_cast<double>(m)) + 1e-9));
    std::vector<int> t0s, t1s, t2s;
    for (int dz = -R; dz <= R; ++dz)
      for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx)
          if (dz * dz + dy * dy + dx * dx == m) {
            t0s.push_back(dz);
            t1s.push_back(dy);
            t2s.push_back(dx);
          }
    const int nt = static_cast<int>(t0s.size());
    if (nt > kMaxTie || R > kMaxTieR || (kTieTY + 2 * R) * (kTieTX + 2 * R) > kTieStage * kTieTX * kTieTY) {   // outside the mask / ring capacity: keep the stencil sweep
      delete B;
      return nullptr;
    }
    tg.R = R;
    tg.ntie = nt;
    tg.ngroup = 0;
    for (int k = 0; k < nt; ++k) {   // t0s is sorted (dz outermost)
      if (tg.ngroup == 0 || tg.t0[tg.ngroup - 1] != t0s[k]) {
        tg.t0[tg.ngroup] = t0s[k];
        tg.beg[tg.ngroup] = k;
        ++tg.ngroup;
      }
      tg.t1[k] = t1s[k];
      tg.t2[k] = t2s[k];
      tg.off[k] = t1s[k] * (kTieTX + 2 * R) + t2s[k];
    }
    tg.beg[tg.ngroup] = nt;
    int q = 0;
    for (int gi = 0; gi < tg.ngroup; ++gi) {
      int a = std::abs(tg.t0[gi]), b = q;
      while (b) { const int t = a % b; a = b; b = t; }
      q = a;
    }
    tg.q = q == 0 ? 1 : q;
    const size_t ring = sizeof(double2) * (2 * R / tg.q + 2) * ((kTieTY + 2 * R) * (kTieTX + 2 * R) + 1);
    if (ring > 227 * 1024) {   // the plane ring does not fit in shared memory: keep the stencil sweep
      delete B;
      return nullptr;
    }
    B->ntie = nt;
    B->tie_m = m;
    B->tie_w = std::pow(static_cast<double>(m), -0.5 * alpha);
    B->tie_thr = sqrt_threshold_host(P.delta0);
  }
  B->twx = upload_on(twiddles3(lx), P.stream);
  B->twy = B->twx;
  double* dw = upload_on(w, P.stream);
  double* cx = upload_on(costab(lx), P.stream);
  NLG_CUDA(cudaMalloc(&B->g, sizeof(double) * static_cast<size_t>(lx) * lx * G));
  NLG_CUDA(cudaMalloc(&B->z, sizeof(double2) * static_cast<size_t>(n_in) * lx * lx));
  NLG_CUDA(cudaMalloc(&B->z2, sizeof(double2) * static_cast<size_t>(n_in) * lx * lx));
  {
    const char* te = std::getenv("NLG_F3_TMA");
    const char* pe = std::getenv("NLG_F3_PERS");
    const bool want_pers = pe && std::atoi(pe) >= 1;
    if (const char* pc = std::getenv("NLG_F3_PERS_CTAS")) B->pers_ctas = std::max(1, std::atoi(pc));
    if ((te && std::atoi(te) == 1) || want_pers) {
      int br = 1;
      for (int d = 1; d <= 256 && d <= lx; ++d)
        if (lx % d == 0) br = d;
      B->tma_br = br;
      double2* zo = B->z2 + static_cast<size_t>(B->o0) * lx * lx;
      B->tma = encode_cols_map(&B->pb_in, B->z, lx, lx, n, n_in, br) &&
               encode_cols_map(&B->pb_out, B->z, lx, lx, lx, n_in, br) &&
               encode_cols_map(&B->pd_in, zo, lx, lx, lx, B->rows_out, br) &&
               encode_cols_map(&B->pd_out, zo, lx, lx, n, B->rows_out, br);
      B->pers = B->tma && want_pers;
      B->tma = B->tma && te && std::atoi(te) == 1;
    }
  }
  const double scale = 1.0 / (static_cast<double>(lx) * lx);
  f3_spectrum<<<static_cast<unsigned>((static_cast<int64_t>(lx) * lx + 255) / 256), 256, 0, P.stream>>>(
      dw, rf, lx, lx, cx, cx, scale, B->g);
  NLG_CUDA(cudaGetLastError());
  NLG_CUDA(cudaStreamSynchronize(P.stream));
  cudaFree(dw);
  cudaFree(cx);
  if (B->ntie > 0) {
    const bool wide = B->ntie > 32;
    const size_t nmask = static_cast<size_t>(B->rows_out) * n * n;
    NLG_CUDA(cudaMalloc(&B->tie_mask, nmask * (wide ? 8 : 4)));
    TieArgs t = tie_args(P, *B);
    const dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((n + 7) / 8),
                    static_cast<unsigned>(B->rows_out));
    if (wide) f3_tie_mask<uint64_t><<<grid, dim3(32, 8), 0, P.stream>>>(t, static_cast<uint64_t*>(B->tie_mask));
    else f3_tie_mask<uint32_t><<<grid, dim3(32, 8), 0, P.stream>>>(t, static_cast<uint32_t*>(B->tie_mask));
    NLG_CUDA(cudaGetLastError());
    NLG_CUDA(cudaStreamSynchronize(P.stream));
    {
      constexpr TieSet kD = make_ties(kTieFixedM, true);
      const char* te = std::getenv("NLG_TIES_TMA");
      B->tie_tma = !(te && std::atoi(te) == 0) && B->tie_m == kTieFixedM && B->ntie <= 32 && n % 2 == 0;
      if (B->tie_tma && P.d_kappa) B->tie_tma = encode_window_map(&B->tmk, P.d_kappa, n, n_in, kD.R);
      for (const void* f : {reinterpret_cast<const void*>(f3_ties_tma<true>), reinterpret_cast<const void*>(f3_ties_tma<false>)})
        NLG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));   // + static mbarriers
    }
    for (const void* f : {reinterpret_cast<const void*>(f3_ties<0, true, uint32_t>), reinterpret_cast<const void*>(f3_ties<0, false, uint32_t>),
                          reinterpret_cast<const void*>(f3_ties<0, true, uint64_t>), reinterpret_cast<const void*>(f3_ties<0, false, uint64_t>),
                          reinterpret_cast<const void*>(f3_ties<kTieFixedM, true, uint32_t>),
                          reinterpret_cast<const void*>(f3_ties<kTieFixedM, false, uint32_t>)})
      NLG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  }
#define NLG_F3_CASE(N) \
  if (lx == N) f3_attr<N>(rf);
  NLG_F3_L(NLG_F3_CASE)
#undef NLG_F3_CASE
  return B;
}

namespace {

F3Args apply_args(Plan& P, BoxFft& B, const double* u, const double* scale, double scale0, const double* diag,
                  double* out) {
  F3Args a = args_of(P, B);
  a.u = u;
  a.scale = scale;
  a.scale0 = scale0;
  a.diag = diag;
  a.out = out;
  a.ab = B.ntie > 0;   // with a tie band the tie pass writes out
  return a;
}

}  // namespace

// PA + PB on input planes [p0, p1)
void boxfft_in(Plan& P, BoxFft& B, const double* u, int64_t p0, int64_t p1, cudaStream_t s) {
  if (p1 <= p0) return;
  F3Args a = apply_args(P, B, u, nullptr, 0.0, nullptr, nullptr);
  a.p0 = p0;
  a.p1 = p1;
  const int lx = B.lx;
  cudaEvent_t ev;
  stage_begin(P, s, kStBoxPA, &ev);
#define NLG_F3_CASE(N) \
  if (lx == N) launch_rows<N>(a, false, (p1 - p0) * B.n, s);
  NLG_F3_L(NLG_F3_CASE)
#undef NLG_F3_CASE
  stage_end(P, s, kStBoxPA, ev, 1);
  stage_begin(P, s, kStBoxPB, &ev);
#define NLG_F3_CASE(N) \
  if (lx == N) { if (B.pers) launch_cols_pers<N>(B, a, false, p1 - p0, s); else if (B.tma) launch_cols_tma<N>(B, a, false, p1 - p0, s); else launch_cols<N>(a, B.cols, false, p1 - p0, s); }
  NLG_F3_L(NLG_F3_CASE)
#undef NLG_F3_CASE
  stage_end(P, s, kStBoxPB, ev, 1);
}

// PC, PD, PE and the tie pass on output planes [q0, q1) (needs PB done on the
// input planes up to q1 + r_f)
void boxfft_out(Plan& P, BoxFft& B, const double* u, const double* scale, double scale0, const double* diag,
                double* out, int64_t q0, int64_t q1, cudaStream_t s, int parts) {
  if (q1 <= q0) return;
  F3Args a = apply_args(P, B, u, scale, scale0, diag, out);
  a.p0 = q0;
  a.p1 = q1;
  const int lx = B.lx;
  cudaEvent_t ev;
  if (parts & 1) {
    stage_begin(P, s, kStBoxPC, &ev);
    launch_zstencil(a, s);
    stage_end(P, s, kStBoxPC, ev, 1);
  }
  if (parts & 2) {
    stage_begin(P, s, kStBoxPD, &ev);
#define NLG_F3_CASE(N) \
  if (lx == N) { if (B.pers) launch_cols_pers<N>(B, a, true, q1 - q0, s); else if (B.tma) launch_cols_tma<N>(B, a, true, q1 - q0, s); else launch_cols<N>(a, B.cols, true, q1 - q0, s); }
    NLG_F3_L(NLG_F3_CASE)
#undef NLG_F3_CASE
    stage_end(P, s, kStBoxPD, ev, 1);
  }
  if (parts & 4) {
    stage_begin(P, s, kStBoxPE, &ev);
#define NLG_F3_CASE(N) \
  if (lx == N) launch_rows<N>(a, true, (q1 - q0) * B.n, s);
    NLG_F3_L(NLG_F3_CASE)
#undef NLG_F3_CASE
    stage_end(P, s, kStBoxPE, ev, 1);
  }
  if (B.ntie > 0 && (parts & 8)) {
    stage_begin(P, s, kStBoxTie, &ev);
    TieArgs t = tie_args(P, B);
    t.u = u;
    t.scale = scale;
    t.scale0 = scale0;
    t.out = out;
    t.diag = diag;
    t.zlo = P.geom.row_begin + q0;
    t.zhi = P.geom.row_begin + q1;
    const bool wide = B.ntie > 32;
    const bool fixed = B.tie_m == kTieFixedM && !wide;
    constexpr TieSet kDense = make_ties(kTieFixedM, true);
    const int R = fixed ? kDense.R : B.tg.R, q = fixed ? kDense.q : B.tg.q, NS = 2 * R / q + 1;
    const size_t sb = sizeof(double2) * ((NS + 1) * ((kTieTY + 2 * R) * (kTieTX + 2 * R) + 1) +
                                         (fixed ? 2 * (R * (kTieTX + 2 * R) + R) + 16 : 0));
    const dim3 grid(static_cast<unsigned>((B.n + kTieTX - 1) / kTieTX), static_cast<unsigned>((B.n + kTieTY - 1) / kTieTY),
                    static_cast<unsigned>((q1 - q0 + kTieZC - 1) / kTieZC * q));
    const dim3 blk(kTieTX, kTieTY);
    if (fixed && B.tie_tma && (B.tmu_base == u || encode_window_map(&B.tmu, u, B.n, B.n_in, kDense.R))) {
      B.tmu_base = u;
      constexpr int NR = 2 * kDense.R / kDense.q + 3;
      const size_t sbt = sizeof(double) * NR * (P.d_kappa ? 2 : 1) * (kTieTY + 2 * kDense.R) * (kTieTX + 2 * kDense.R);
      if (P.d_kappa) f3_ties_tma<true><<<grid, blk, sbt, s>>>(B.tmu, B.tmk, t);
      else f3_ties_tma<false><<<grid, blk, sbt, s>>>(B.tmu, B.tmk, t);
    } else if (wide) {
      if (P.d_kappa) f3_ties<0, true, uint64_t><<<grid, blk, sb, s>>>(t);
      else f3_ties<0, false, uint64_t><<<grid, blk, sb, s>>>(t);
    } else if (fixed) {
      if (P.d_kappa) f3_ties<kTieFixedM, true, uint32_t><<<grid, blk, sb, s>>>(t);
      else f3_ties<kTieFixedM, false, uint32_t><<<grid, blk, sb, s>>>(t);
    } else {
      if (P.d_kappa) f3_ties<0, true, uint32_t><<<grid, blk, sb, s>>>(t);
      else f3_ties<0, false, uint32_t><<<grid, blk, sb, s>>>(t);
    }
    stage_end(P, s, kStBoxTie, ev, 1);
  }
}

void boxfft_apply(Plan& P, BoxFft& B, const double* u, const double* scale, double scale0, const double* diag,
                  double* out, cudaStream_t s) {
  // NLG_F3_CHUNK=k (planes, read once): PA -> PB and PD -> PE run chunk by chunk so the
  // second pass of each pair finds its input in L2 (a plane of Z is ~10 MB at L = 800)
  static const int chunk = [] { const char* e = std::getenv("NLG_F3_CHUNK"); return e ? std::atoi(e) : 0; }();
  if (chunk <= 0) {
    boxfft_in(P, B, u, 0, B.n_in, s);
    boxfft_out(P, B, u, scale, scale0, diag, out, 0, B.rows_out, s);
    return;
  }
  for (int64_t p0 = 0; p0 < B.n_in; p0 += chunk) boxfft_in(P, B, u, p0, std::min<int64_t>(p0 + chunk, B.n_in), s);
  boxfft_out(P, B, u, scale, scale0, diag, out, 0, B.rows_out, s, 1);
  for (int64_t q0 = 0; q0 < B.rows_out; q0 += chunk)
    boxfft_out(P, B, u, scale, scale0, diag, out, q0, std::min<int64_t>(q0 + chunk, B.rows_out), s, 2 | 4);
  boxfft_out(P, B, u, scale, scale0, diag, out, 0, B.rows_out, s, 8);
}

int boxfft_launches(const BoxFft& B) { return 5 + (B.ntie > 0 ? 1 : 0); }
int boxfft_length(const BoxFft& B) { return B.lx; }

void boxfft_free(BoxFft* B) {
  if (!B) return;
  for (void* p : {static_cast<void*>(B->twx), static_cast<void*>(B->g),
                  static_cast<void*>(B->z), static_cast<void*>(B->z2), B->tie_mask})
    cudaFree(p);
  delete B;
}

}  // namespace nlg
