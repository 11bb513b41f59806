// paper_1905_08375_b200/csrc/fft.cuh — four-step fp64 FFT convolution for the
// 1-D fixed-window far field (expsum FFT mode), with the field packing, the
// spectrum product fused into its three HBM passes.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nlg {

// L = N1 * N2 (N2 = 2^b rows, N1 = 2^a {1,3,9} columns); element x of the
// signal is (n1, n2) = (x / N2, x % N2), frequency k = k1 + N1 k2.
struct FourStep {
  int64_t L = 0;
  int n1 = 0, n2 = 0;
  double2* tw1 = nullptr;    // [N1] exp(-2 pi i t / N1)
  double2* tw2 = nullptr;    // [N2] exp(-2 pi i t / N2)
  double2* twa = nullptr;    // [L / 4096 + 1] exp(-2 pi i 4096 a / L)
  double2* twb = nullptr;    // [4096] exp(-2 pi i b / L)
  double* krp = nullptr;     // [N1][N2] kernel spectrum / L at k1 + N1 k2
  int64_t rows_grid = 0;     // P2 persistent grid (0: one CTA per row)
};

// Plan for length L, or false when L has no supported split (the caller then
// runs the cuFFT path).
bool fourstep_plan(int64_t L, FourStep& F);
// Smallest L >= m with the preferred 4096-row split and >= 256 columns (0 when
// another split or the cuFFT path is forced through NLG_FS_ROWS).
int64_t fourstep_length(int64_t m);
// Device tables; kr = real kernel spectrum in natural order (length L).
void fourstep_setup(FourStep& F, const double* kr, cudaStream_t s);
void fourstep_free(FourStep& F);
// z <- row spectra product, from u (+ kappa u) (passes 1 and 2)
void fourstep_forward_product(const FourStep& F, const double* u, const double* kappa, int64_t n_in, double2* z,
                              cudaStream_t s);
// inverse column pass alone: z <- (conv u, conv kappa u) in signal order
void fourstep_inverse(const FourStep& F, double2* z, cudaStream_t s);
// the two halves of fourstep_forward_product (per-kernel timing)
void fourstep_cols_forward(const FourStep& F, const double* u, const double* kappa, int64_t n_in, double2* z,
                           cudaStream_t s);
void fourstep_rows_product(const FourStep& F, double2* z, cudaStream_t s);

}  // namespace nlg
