// paper_1905_08375_b200/csrc/fft.cu — four-step fp64 FFT convolution (expsum
// FFT mode).
//
// The fixed-window far field is conv(f, K) for f = u + i kappa u (two real
// fields in one complex signal) and the real symmetric window kernel K. With
// L = N1 N2, x = N2 n1 + n2 and k = k1 + N1 k2 the transform splits into
// column FFTs (length N1), a twiddle W_L^{n2 k1} and row FFTs (length N2). The
// whole convolution runs in three HBM passes:
//   P1 fs_cols_fwd : load u, kappa (the packing), column FFTs, twiddle -> z
//   P2 fs_rows     : row FFT, x K^/L, conj, row FFT (the inverse row step by
//                    the conjugate identity), one CTA per row in shared memory
//   P3 fs_cols_inv : twiddle, column FFTs, conj -> conv (in z, signal order)
// Every FFT is a self-sorting mixed-radix Stockham transform in shared memory
// (radix 2/3/4/8 butterflies held in registers between two barriers).
// Against the cuFFT chain (pack, 3 + 3 passes, spectrum product) this moves
// ~0.55 GB instead of ~1.2 GB per apply at N = 2^22; all three passes run on
// the side stream, overlapping the exponential-sum scans.
#include "fft.cuh"

#include <cmath>
#include <cstdlib>
#include <vector>

#include "plan.hpp"
#include "stockham.cuh"

namespace nlg {
namespace {

using namespace stockham;

constexpr int kFsEl = 8;         // elements per thread per stage (register budget)
#ifndef NLG_FS_WIDE
#define NLG_FS_WIDE 0             // experiment: 8 columns per CTA beyond N1 = 768 (16 elements per thread, one CTA per
                                  // SM): 64-byte u pieces, but 70 vs 60 us per column pass at cfg1 (0.448 vs 0.426 ms)
#endif
#ifndef NLG_FS_KRP_PREFETCH
#define NLG_FS_KRP_PREFETCH 0     // K^ row staged by cp.async (208 KB CTAs: no co-residence with the scans)
#endif
constexpr int kFsTwB = 4096;     // four-step twiddle split: W^P = A[P / 4096] B[P % 4096]

struct FsDev {
  int n1, n2;
  const double2* tw1;
  const double2* tw2;
  const double2* twa;
  const double2* twb;
  const double* krp;
};

__device__ __forceinline__ double2 four_tw(const FsDev& d, int p) {   // W_L^p, 0 <= p < L
  return cmul(__ldg(d.twa + (p >> 12)), __ldg(d.twb + (p & (kFsTwB - 1))));
}

// column passes: C columns per CTA (8: 128-byte row pieces; 4 beyond N1 = 768
// to stay within 576 threads), T threads cover the N1 * C elements, kFsEl each
template <int N1>
__host__ __device__ constexpr int cols_c() { return N1 <= 768 || NLG_FS_WIDE ? 8 : 4; }
template <int N1>
__host__ __device__ constexpr int cols_el() { return N1 * cols_c<N1>() > 1024 * kFsEl ? 2 * kFsEl : kFsEl; }
template <int N1>
__host__ __device__ constexpr int cols_threads() { return (N1 * cols_c<N1>() + cols_el<N1>() - 1) / cols_el<N1>(); }
template <int N1>
__host__ __device__ constexpr int cols_ctas() { return cols_el<N1>() > kFsEl ? 1 : 2; }

// P1: columns c0..c0+7, x = N2 n1 + n2 -> z[k1][n2] = W^{n2 k1} FFT_N1(f)[k1]
template <int N1, bool KW>
__global__ void __launch_bounds__(cols_threads<N1>(), cols_ctas<N1>()) fs_cols_fwd(const __grid_constant__ FsDev d,
                                                                    const double* __restrict__ u,
                                                                    const double* __restrict__ kappa, int64_t n_in,
                                                                    double2* __restrict__ z) {
  constexpr int T = cols_threads<N1>(), C = cols_c<N1>();
  extern __shared__ double2 fsm[];
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * C;
  auto ld = [&](int n1, int c) {
    const int64_t x = static_cast<int64_t>(n1) * d.n2 + c0 + c;
    if (x >= n_in) return make_double2(0.0, 0.0);
    const double a = __ldg(u + x);
    return make_double2(a, KW ? a * __ldg(kappa + x) : 0.0);
  };
  auto st = [&](int base, int stride, int c, auto& v) {   // k1 = base + r stride
    constexpr int R = sizeof(v) / sizeof(v[0]);
    const int n2 = c0 + c;
    double2 w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) w[r] = four_tw(d, n2 * (base + r * stride));
#pragma unroll
    for (int r = 0; r < R; ++r) z[static_cast<int64_t>(base + r * stride) * d.n2 + n2] = cmul(v[r], w[r]);
  };
  fs_fft<false, N1, 1, N1, C, T, false>(fsm, d.tw1, tid, ld, st);
}

// P2: one row k1: forward FFT, x K^[k1 + N1 k2] / L, conjugate, forward FFT.
// The last forward stage (thread j holds X[j + r N/R]) and the first stage of
// the second transform (reads j + r N/R) share their elements: the spectrum
// product happens in registers between the two butterflies.
template <int N2>
__global__ void __launch_bounds__(N2 / rows_el<N2>(), (N2 / rows_el<N2>() <= 512 && N2 < 8192) ? 2 : 1)
    fs_rows(const __grid_constant__ FsDev d, double2* __restrict__ z) {
  constexpr int T = N2 / rows_el<N2>();
  constexpr int R = rows_el<N2>();      // first = last radix of the row plan
  constexpr int nq = N2 / R;
  static_assert(nq == T, "one butterfly per thread in the fused stage");
  extern __shared__ double2 fsm[];
  double* skr = reinterpret_cast<double*>(fsm + N2 + N2 / 8);   // the row of K^ / L, prefetched
  const int tid = threadIdx.x;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * N2;
#if NLG_FS_KRP_PREFETCH
#pragma unroll
  for (int it = 0; it < N2 / T; ++it) {
    const int q = tid + it * T;
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(skr + q));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(d.krp + row + q) : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
#endif
  auto ld = [&](int e, int) { return z[row + e]; };
  auto none = [&](int, int, int, auto&) {};
  // forward transform up to (not including) its last stage
  fs_fft<true, N2, 1, N2 / R, 1, T, true>(fsm, d.tw2, tid, ld, none);
  {
    // fused: last forward stage (Ns = N2 / R), product, first stage of the second transform
    constexpr int Ns = N2 / R;
    const int j = tid, k = j;           // j < Ns
#if NLG_FS_KRP_PREFETCH
    asm volatile("cp.async.wait_all;\n" ::: "memory");   // own K^ loads; the barrier below publishes all
#endif
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = fsm[sidx<true>(j + r * nq)];
    __syncthreads();
    if (k > 0) {
      const double2 w = __ldg(d.tw2 + k * (N2 / (Ns * R)));
      double2 wr = w;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        v[r] = cmul(v[r], wr);
        if (r + 1 < R) wr = cmul(wr, w);
      }
    }
    Dft<R>::run(v);
#pragma unroll
    for (int r = 0; r < R; ++r) {       // X[j + r Ns]: x K^ / L, conjugate
#if NLG_FS_KRP_PREFETCH
      const double kk = skr[j + r * Ns];
#else
      const double kk = __ldg(d.krp + row + j + r * Ns);
#endif
      v[r] = make_double2(v[r].x * kk, -v[r].y * kk);
    }
    Dft<R>::run(v);                     // first stage of the second transform (Ns = 1)
#pragma unroll
    for (int r = 0; r < R; ++r) fsm[sidx<true>(j * R + r)] = v[r];
    __syncthreads();
  }
  auto st = [&](int base, int stride, int, auto& v) {
    constexpr int RR = sizeof(v) / sizeof(v[0]);
#pragma unroll
    for (int r = 0; r < RR; ++r) z[row + base + r * stride] = v[r];
  };
  fs_fft<true, N2, R, N2, 1, T, true>(fsm, d.tw2, tid, ld, st);
}

// P2, persistent: CTAs loop over rows (grid = resident CTAs) and prefetch the
// next row's first-stage inputs and K^ values into registers while the
// current row is in its later stages, so HBM stays busy while a CTA computes
// (the one-row kernel above loads, computes and stores in series).
template <int N2>
__global__ void __launch_bounds__(N2 / rows_el<N2>(), 1)
    fs_rows_pp(const __grid_constant__ FsDev d, double2* __restrict__ z, int nrows) {
  constexpr int T = N2 / rows_el<N2>();
  constexpr int R = rows_el<N2>();
  constexpr int nq = N2 / R;
  static_assert(nq == T, "one butterfly per thread in the first and fused stages");
  extern __shared__ double2 fsm[];
  const int tid = threadIdx.x;
  double2 pre[R];
  double kpre[R];
  auto fetch_z = [&](int rw) {
    if (rw < nrows) {
      const double2* src = z + static_cast<int64_t>(rw) * N2 + tid;
#pragma unroll
      for (int r = 0; r < R; ++r) pre[r] = src[r * nq];
    }
  };
  auto fetch_k = [&](int rw) {
    if (rw < nrows) {
      const double* src = d.krp + static_cast<int64_t>(rw) * N2 + tid;
#pragma unroll
      for (int r = 0; r < R; ++r) kpre[r] = __ldg(src + r * nq);
    }
  };
  int rw = blockIdx.x;
  fetch_z(rw);
  fetch_k(rw);
  for (; rw < nrows; rw += gridDim.x) {
    const int64_t row = static_cast<int64_t>(rw) * N2;
    // first stage from the prefetched registers: element e = tid + r nq is pre[r]
    auto ld = [&](int e, int) { return pre[(e - tid) / nq]; };
    auto none = [&](int, int, int, auto&) {};
    fs_fft<true, N2, 1, R, 1, T, true>(fsm, d.tw2, tid, ld, none);
    fetch_z(rw + gridDim.x);                                   // next row in flight
    fs_fft<true, N2, R, N2 / R, 1, T, true>(fsm, d.tw2, tid, ld, none);
    {
      constexpr int Ns = N2 / R;
      const int j = tid, k = j;
      double2 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = fsm[sidx<true>(j + r * nq)];
      __syncthreads();
      if (k > 0) {
        const double2 w = __ldg(d.tw2 + k * (N2 / (Ns * R)));
        double2 wr = w;
#pragma unroll
        for (int r = 1; r < R; ++r) {
          v[r] = cmul(v[r], wr);
          if (r + 1 < R) wr = cmul(wr, w);
        }
      }
      Dft<R>::run(v);
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = make_double2(v[r].x * kpre[r], -v[r].y * kpre[r]);   // K^[j + r Ns]
      fetch_k(rw + gridDim.x);
      Dft<R>::run(v);
#pragma unroll
      for (int r = 0; r < R; ++r) fsm[sidx<true>(j * R + r)] = v[r];
      __syncthreads();
    }
    auto st = [&](int base, int stride, int, auto& v) {
      constexpr int RR = sizeof(v) / sizeof(v[0]);
#pragma unroll
      for (int r = 0; r < RR; ++r) z[row + base + r * stride] = v[r];
    };
    fs_fft<true, N2, R, N2, 1, T, true>(fsm, d.tw2, tid, ld, st);
    __syncthreads();                                           // last stage's shared reads before the next row
  }
}

// P3: columns: conv(x) = conj(FFT_N1(W^{n2 k1} z[k1][n2]))[n1] -> z[x] = (conv u, conv kappa u),
// in place (a CTA reads and writes only its own columns)
template <int N1>
__global__ void __launch_bounds__(cols_threads<N1>(), cols_ctas<N1>()) fs_cols_inv(const __grid_constant__ FsDev d,
                                                                          double2* z) {
  constexpr int T = cols_threads<N1>(), C = cols_c<N1>();
  extern __shared__ double2 fsm[];
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * C;
  auto ld = [&](int k1, int c) {
    const int n2 = c0 + c;
    return cmul(z[static_cast<int64_t>(k1) * d.n2 + n2], four_tw(d, n2 * k1));
  };
  auto st = [&](int base, int stride, int c, auto& v) {
    constexpr int R = sizeof(v) / sizeof(v[0]);
#pragma unroll
    for (int r = 0; r < R; ++r)
      z[static_cast<int64_t>(base + r * stride) * d.n2 + c0 + c] = make_double2(v[r].x, -v[r].y);
  };
  fs_fft<false, N1, 1, N1, C, T, false>(fsm, d.tw1, tid, ld, st);
}

__global__ void fs_permute(const double* __restrict__ kr, double* __restrict__ krp, int n1, int n2, double inv_l) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;   // k1 * N2 + k2
  if (q >= static_cast<int64_t>(n1) * n2) return;
  const int64_t k1 = q / n2, k2 = q % n2;
  krp[q] = kr[k1 + n1 * k2] * inv_l;
}

FsDev dev_of(const FourStep& F) {
  FsDev d;
  d.n1 = F.n1;
  d.n2 = F.n2;
  d.tw1 = F.tw1;
  d.tw2 = F.tw2;
  d.twa = F.twa;
  d.twb = F.twb;
  d.krp = F.krp;
  return d;
}

// supported column lengths 2^a {1, 3, 9} in [64, 1536], plus 320 and 1080 (radix-5 stages:
// tighter lengths for cfg1 and its 4- and 8-way slabs)
#define NLG_FS_N1(X) \
  X(64) X(72) X(96) X(128) X(144) X(192) X(256) X(288) X(320) X(384) X(512) X(576) X(768) X(1024) \
  X(1080) X(1152) X(1536)

template <int N1>
size_t cols_smem() { return sizeof(double2) * N1 * cols_c<N1>(); }
size_t rows_smem(int n2) { return sizeof(double2) * (n2 + n2 / 8) + (NLG_FS_KRP_PREFETCH ? sizeof(double) * n2 : 0); }

template <int N1>
void cols_attr() {
  for (const void* f : {reinterpret_cast<const void*>(fs_cols_fwd<N1, true>), reinterpret_cast<const void*>(fs_cols_fwd<N1, false>),
                        reinterpret_cast<const void*>(fs_cols_inv<N1>)})
    NLG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cols_smem<N1>())));
}

template <int N1>
void cols_fwd(const FsDev& d, const double* u, const double* kappa, int64_t n_in, double2* z, cudaStream_t s) {
  const unsigned g = static_cast<unsigned>(d.n2 / cols_c<N1>());
  if (kappa) fs_cols_fwd<N1, true><<<g, cols_threads<N1>(), cols_smem<N1>(), s>>>(d, u, kappa, n_in, z);
  else fs_cols_fwd<N1, false><<<g, cols_threads<N1>(), cols_smem<N1>(), s>>>(d, u, kappa, n_in, z);
}

template <int N1>
void cols_inv(const FsDev& d, double2* z, cudaStream_t s) {
  const unsigned g = static_cast<unsigned>(d.n2 / cols_c<N1>());
  fs_cols_inv<N1><<<g, cols_threads<N1>(), cols_smem<N1>(), s>>>(d, z);
}


bool n1_supported(int64_t n1) {
#define NLG_FS_CASE(N) if (n1 == N) return true;
  NLG_FS_N1(NLG_FS_CASE)
#undef NLG_FS_CASE
  return false;
}

std::vector<double2> twiddles(int64_t n, int64_t count, int64_t step) {   // exp(-2 pi i step t / n)
  std::vector<double2> t(static_cast<size_t>(count));
  const long double pi2 = 2.0L * std::acos(-1.0L);
  for (int64_t i = 0; i < count; ++i) {
    const long double a = pi2 * static_cast<long double>((step * i) % n) / static_cast<long double>(n);
    t[i] = make_double2(static_cast<double>(std::cos(a)), static_cast<double>(-std::sin(a)));
  }
  return t;
}


}  // namespace

#ifndef NLG_FS_ROWS_FIRST
#define NLG_FS_ROWS_FIRST 4096   // preferred row length when several splits exist (measured, cfg1:
                                 // 4096 x 1152 beats 8192 x 576 by 3%: two row CTAs per SM)
#endif

// Only the preferred 4096-row split with columns of at least 256 (measured:
// 1080 x 4096 for cfg1 and 320 x 4096 for its 4-way slabs beat the next
// 2^a {1,3,9} length; a 2048-row or a 180-column split does not).
int64_t fourstep_length(int64_t m) {
  const char* env = std::getenv("NLG_FS_ROWS");
  if (env && std::atoi(env) != NLG_FS_ROWS_FIRST) return 0;   // forced splits / cuFFT: the 2^a {1,3,9} lengths
  const int64_t n2 = NLG_FS_ROWS_FIRST;
  int64_t best = 0;
#define NLG_FS_CASE(N) \
  if (N >= 256 && N * n2 >= m && (best == 0 || N * n2 < best)) best = N * n2;
  NLG_FS_N1(NLG_FS_CASE)
#undef NLG_FS_CASE
  return best;
}

bool fourstep_plan(int64_t L, FourStep& F) {
  // NLG_FS_ROWS (environment, read at plan time): preferred row length, for tests
  const char* env = std::getenv("NLG_FS_ROWS");
  const int first = env ? std::atoi(env) : NLG_FS_ROWS_FIRST;
  if (first == 0) return false;                               // force the cuFFT path
  const int order[3] = {first, first == 4096 ? 8192 : 4096, first == 2048 ? 8192 : 2048};
  for (int n2 : order) {
    if (L % n2 || !n1_supported(L / n2)) continue;
    F.L = L;
    F.n1 = static_cast<int>(L / n2);
    F.n2 = n2;
    return true;
  }
  return false;
}

void fourstep_setup(FourStep& F, const double* kr, cudaStream_t s) {
  F.tw1 = upload_on(twiddles(F.n1, F.n1, 1), s);
  F.tw2 = upload_on(twiddles(F.n2, F.n2, 1), s);
  F.twa = upload_on(twiddles(F.L, F.L / kFsTwB + 1, kFsTwB), s);
  F.twb = upload_on(twiddles(F.L, kFsTwB, 1), s);
  NLG_CUDA(cudaMalloc(&F.krp, sizeof(double) * F.L));
  fs_permute<<<static_cast<unsigned>((F.L + 255) / 256), 256, 0, s>>>(kr, F.krp, F.n1, F.n2,
                                                                      1.0 / static_cast<double>(F.L));
  NLG_CUDA(cudaGetLastError());
#define NLG_FS_CASE(N) \
  if (F.n1 == N) cols_attr<N>();
  NLG_FS_N1(NLG_FS_CASE)
#undef NLG_FS_CASE
  for (const void* f : {reinterpret_cast<const void*>(fs_rows<2048>), reinterpret_cast<const void*>(fs_rows<4096>),
                        reinterpret_cast<const void*>(fs_rows<8192>)})
    NLG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rows_smem(8192))));   // 208 KB
  for (const void* f : {reinterpret_cast<const void*>(fs_rows_pp<2048>), reinterpret_cast<const void*>(fs_rows_pp<4096>),
                        reinterpret_cast<const void*>(fs_rows_pp<8192>)})
    NLG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rows_smem(8192))));
  // persistent rows: one resident CTA wave looping over the rows, selected by
  // NLG_FS_PERSIST=1 at plan time (cfg1: 71 vs 75 us isolated, no change
  // inside the overlapped apply: 0.438 vs 0.437 ms; default one CTA per row)
  const char* pe = std::getenv("NLG_FS_PERSIST");
  F.rows_grid = 0;
  if (pe && std::atoi(pe) == 1) {
    int dev = 0, sms = 0, per = 0;
    NLG_CUDA(cudaGetDevice(&dev));
    NLG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t rp = sizeof(double2) * (F.n2 + F.n2 / 8);
    const void* f = F.n2 == 8192 ? reinterpret_cast<const void*>(fs_rows_pp<8192>)
                    : (F.n2 == 4096 ? reinterpret_cast<const void*>(fs_rows_pp<4096>)
                                    : reinterpret_cast<const void*>(fs_rows_pp<2048>));
    const int thr = F.n2 == 8192 ? 8192 / rows_el<8192>() : (F.n2 == 4096 ? 4096 / rows_el<4096>() : 2048 / rows_el<2048>());
    NLG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, thr, rp));
    F.rows_grid = std::min<int64_t>(F.n1, static_cast<int64_t>(std::max(per, 1)) * sms);
  }
}

void fourstep_free(FourStep& F) {
  for (double2* p : {F.tw1, F.tw2, F.twa, F.twb}) cudaFree(p);
  cudaFree(F.krp);
  F = FourStep{};
}

void fourstep_cols_forward(const FourStep& F, const double* u, const double* kappa, int64_t n_in, double2* z,
                           cudaStream_t s) {
  const FsDev d = dev_of(F);
#define NLG_FS_CASE(N) \
  if (F.n1 == N) cols_fwd<N>(d, u, kappa, n_in, z, s);
  NLG_FS_N1(NLG_FS_CASE)
#undef NLG_FS_CASE
}

void fourstep_rows_product(const FourStep& F, double2* z, cudaStream_t s) {
  const FsDev d = dev_of(F);
  const size_t rs = rows_smem(F.n2);
  if (F.rows_grid > 0) {   // persistent rows (register prefetch of the next row)
    const unsigned g = static_cast<unsigned>(F.rows_grid);
    const size_t rp = sizeof(double2) * (F.n2 + F.n2 / 8);
    if (F.n2 == 8192) fs_rows_pp<8192><<<g, 8192 / rows_el<8192>(), rp, s>>>(d, z, F.n1);
    else if (F.n2 == 4096) fs_rows_pp<4096><<<g, 4096 / rows_el<4096>(), rp, s>>>(d, z, F.n1);
    else fs_rows_pp<2048><<<g, 2048 / rows_el<2048>(), rp, s>>>(d, z, F.n1);
    return;
  }
  if (F.n2 == 8192) fs_rows<8192><<<F.n1, 8192 / rows_el<8192>(), rs, s>>>(d, z);
  else if (F.n2 == 4096) fs_rows<4096><<<F.n1, 4096 / rows_el<4096>(), rs, s>>>(d, z);
  else fs_rows<2048><<<F.n1, 2048 / rows_el<2048>(), rs, s>>>(d, z);
}

void fourstep_forward_product(const FourStep& F, const double* u, const double* kappa, int64_t n_in, double2* z,
                              cudaStream_t s) {
  fourstep_cols_forward(F, u, kappa, n_in, z, s);
  fourstep_rows_product(F, z, s);
}

void fourstep_inverse(const FourStep& F, double2* z, cudaStream_t s) {
  const FsDev d = dev_of(F);
#define NLG_FS_CASE(N) \
  if (F.n1 == N) cols_inv<N>(d, z, s);
  NLG_FS_N1(NLG_FS_CASE)
#undef NLG_FS_CASE
}


}  // namespace nlg
