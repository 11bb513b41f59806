// paper_1905_08375_b200/csrc/solve.cu — device BLAS-1 for the Krylov consumer
// (solve_dirichlet, reference src/solve.cpp:32-108): deterministic dot
// products (fixed grid, block partials, one final block) with a non-finite
// flag on the operator output (check_finite, solve.cpp:24-28), and the fused
// vector updates of CG / CGNR.
#include "plan.hpp"

namespace nlg {

namespace {

constexpr int kDotBlocks = 296;      // 2 x 148 SMs
constexpr int kDotThreads = 256;

// part[b] = sum over this block's stride of a_i * b_i; bad |= !isfinite(chk_i)
__global__ void __launch_bounds__(kDotThreads) dot_partial(const double* __restrict__ a, const double* __restrict__ b,
                                                           const double* __restrict__ chk, int64_t n,
                                                           double* __restrict__ part, int* __restrict__ bad) {
  double s = 0.0;
  int nonfinite = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kDotThreads + threadIdx.x; i < n;
       i += static_cast<int64_t>(kDotBlocks) * kDotThreads) {
    s = fma(a[i], b[i], s);
    if (chk && !isfinite(chk[i])) nonfinite = 1;
  }
  s = warp_sum(s);
  __shared__ double sw[kDotThreads / 32];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
  if (chk && __syncthreads_or(nonfinite) && threadIdx.x == 0) atomicOr(bad, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kDotThreads / 32; ++w) t += sw[w];
    part[blockIdx.x] = t;
  }
}

__global__ void dot_final(const double* __restrict__ part, double* __restrict__ res) {
  __shared__ double sh[kDotBlocks];
  for (int i = threadIdx.x; i < kDotBlocks; i += blockDim.x) sh[i] = part[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kDotBlocks; ++i) t += sh[i];
    *res = t;
  }
}

// u += alpha p ; r -= alpha ap
__global__ void axpy2_kernel(double* __restrict__ u, double* __restrict__ r, const double* __restrict__ p,
                             const double* __restrict__ ap, double alpha, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  u[i] += alpha * p[i];
  r[i] -= alpha * ap[i];
}

// p = z + beta p
__global__ void xpby_kernel(double* __restrict__ p, const double* __restrict__ z, double beta, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = z[i] + beta * p[i];
}

// x = -x
__global__ void negate_kernel(double* __restrict__ x, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = -x[i];
}

// d = f - x
__global__ void diff_kernel(double* __restrict__ d, const double* __restrict__ f, const double* __restrict__ x,
                            int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) d[i] = f[i] - x[i];
}

unsigned grid_of(int64_t n) { return static_cast<unsigned>((n + 255) / 256); }

}  // namespace

size_t dot_scratch_doubles() { return kDotBlocks + 1; }

void dev_dot(const double* a, const double* b, const double* chk, int64_t n, double* scratch, int* bad,
             cudaStream_t s) {
  dot_partial<<<kDotBlocks, kDotThreads, 0, s>>>(a, b, chk, n, scratch, bad);
  dot_final<<<1, 256, 0, s>>>(scratch, scratch + kDotBlocks);
}

void dev_axpy2(double* u, double* r, const double* p, const double* ap, double alpha, int64_t n, cudaStream_t s) {
  axpy2_kernel<<<grid_of(n), 256, 0, s>>>(u, r, p, ap, alpha, n);
}

void dev_xpby(double* p, const double* z, double beta, int64_t n, cudaStream_t s) {
  xpby_kernel<<<grid_of(n), 256, 0, s>>>(p, z, beta, n);
}

void dev_negate(double* x, int64_t n, cudaStream_t s) { negate_kernel<<<grid_of(n), 256, 0, s>>>(x, n); }

void dev_diff(double* d, const double* f, const double* x, int64_t n, cudaStream_t s) {
  diff_kernel<<<grid_of(n), 256, 0, s>>>(d, f, x, n);
}

}  // namespace nlg
