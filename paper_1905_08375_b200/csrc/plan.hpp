// paper_1905_08375_b200/csrc/plan.hpp — the plan object behind nlg_plan.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/nlgpu.h"
#include "common.cuh"

namespace nlg {

// Error plumbing: CUDA failures become NLG_ECUDA with the CUDA error string.
struct Error {
  nlg_status code;
  std::string msg;
};

#define NLG_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      throw ::nlg::Error{NLG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

// Plan-time uploads, ordered on the plan stream. A pageable source is staged
// before cudaMemcpyAsync returns, so the host buffer may be freed right after;
// kernels on the same stream see the data without a device-wide sync.
template <typename T>
T* upload_on(const T* src, size_t count, cudaStream_t s) {
  T* d = nullptr;
  NLG_CUDA(cudaMalloc(&d, sizeof(T) * (count ? count : 1)));
  if (count) NLG_CUDA(cudaMemcpyAsync(d, src, sizeof(T) * count, cudaMemcpyHostToDevice, s));
  return d;
}
template <typename T>
T* upload_on(const std::vector<T>& v, cudaStream_t s) { return upload_on(v.data(), v.size(), s); }

// 1-D exponential-sum far field (fast method 2).
struct ExpSum {
  int terms = 0;          // M
  int near = 0;           // P: offsets 1..P summed directly
  int64_t dmax = 0;       // largest horizon offset (cells)
  double rel_err = 0.0;   // fitted max relative kernel error on [P+1, dmax]
  std::vector<double> rate;   // t_m  (lambda_m = exp(-t_m))
  std::vector<double> weight; // c_m
};

struct ExpSumState;
struct ScanBuffers;
struct StencilState;
struct BoxFft;

// Optional per-stage CUDA-event timing (nlg_set_profiling / nlg_stage_times).
// With profiling on, every stage is timed on the apply's own stream (side
// streams are folded into it), so the stage times do not overlap and their
// shares add up to the serialized apply.
enum Stage { kStDirect = 0, kStSpanScan, kStSpanEval, kStEsAggregate, kStEsCarry, kStEsMain,
             kStEsCombine, kStStencil, kStEsFft, kStBoxFft, kStBoxTie,
             kStBoxPA, kStBoxPB, kStBoxPC, kStBoxPD, kStBoxPE, kStEsFftP1, kStEsFftP2, kStEsFftP3,
             kNumStages };
struct StageProf {
  bool on = false;
  struct Rec { int stage; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  double ms[kNumStages] = {};
  int64_t launches[kNumStages] = {};
};

struct Plan {
  int family = 0, route = 0, rule = 0, form = 0, exterior = 0, divergence = 0;
  Profile prof{};
  Geom geom{};
  double delta0 = 0, coeff0 = 1, reach = 0, delta_max = 0;
  int64_t n_in = 0, n_out = 0;
  int64_t halo_lo = 0, halo_hi = 0;
  int device = 0;
  int fast_method = 0;
  cudaStream_t stream = nullptr;

  // per-node static fields over the input rows (device)
  double* d_delta = nullptr;
  double* d_coeff = nullptr;
  double* d_kappa = nullptr;

  // KIND 3 direct-sum weight table (direct.cu direct_frac_setup)
  double2* d_wfrac = nullptr;
  int64_t wfrac_len = 0;

  // staging for the host entry points
  double* d_u = nullptr;
  double* d_out = nullptr;
  unsigned long long* d_pairs = nullptr;
  int64_t* d_targets = nullptr;
  int64_t targets_cap = 0;

  // fast method 1 (span prefix sums)
  double* d_pref_hi = nullptr;   // local exclusive prefix, [rows][len]
  double* d_pref_lo = nullptr;
  double* d_seg_hi = nullptr;    // row totals (the prefix at p = len)
  double* d_seg_lo = nullptr;
  ScanBuffers* scan_buf = nullptr;   // look-back state; method 4 moment tables
  int64_t scan_rows = 0, scan_len = 0, scan_nseg = 0;

  // fast method 2 (1-D exponential-sum scans)
  ExpSum es;
  ExpSumState* es_state = nullptr;

  // fast method 3 (2-D/3-D offset-table stencil)
  StencilState* st_state = nullptr;

  // host pipeline of nlg_apply_fast (row chunks: H2D / apply / D2H overlapped)
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  std::vector<cudaEvent_t> pipe_ev;
  bool split_begun = false;   // nlg_apply_fast_dev_begin enqueued the halo-independent part
  int64_t split_lo = 0, split_hi = 0;   // stencil slabs: the output rows begin computed

  int64_t last_pairs = 0;
  int64_t fast_applies = 0;
  int64_t launches = 0;   // kernels launched by this plan (all entry points)
  StageProf sprof;
};

// Stage bracketing: records events when profiling is on; always counts launches.
void stage_begin(Plan& P, cudaStream_t s, int stage, cudaEvent_t* ev);
void stage_end(Plan& P, cudaStream_t s, int stage, cudaEvent_t ev, int nlaunch);

// kernels
void launch_direct(const Plan& P, const double* u, double* out, const int64_t* targets,
                   int64_t ntargets, unsigned long long* pairs, cudaStream_t s);
int direct_kind(const Plan& P);
void direct_frac_setup(Plan& P);
void launch_transpose(const Plan& P, const double* v, double* out, cudaStream_t s);
void launch_assemble(const Plan& P, double* A, int64_t N, cudaStream_t s);
void spans_setup(Plan& P);
void spans_apply(Plan& P, const double* u, double* out, cudaStream_t s);
void spans_free(Plan& P);
void moments_setup(Plan& P, int K);   // fast method 4: 1-D K >= 1 centred moment scans
void moments_apply(Plan& P, const double* u, double* out, cudaStream_t s);
int64_t moments_segment(const Plan& P);
void expsum_setup(Plan& P, const nlg_desc& d);
void expsum_apply(Plan& P, const double* u, double* out, cudaStream_t s);
void expsum_free(Plan& P);
void expsum_fft_info(const Plan& P, int64_t& len, int& rows);
void stencil_setup(Plan& P, const nlg_desc& d);
void stencil_apply(Plan& P, const double* u, double* out, cudaStream_t s);
void stencil_free(Plan& P);
int stencil_launches(const Plan& P);
int stencil_fft_len(const Plan& P);
bool stencil_box(const Plan& P);   // method 3 runs the box FFT mode (brackets its own stages)
void stencil_apply_rows(Plan& P, const double* u, double* out, int64_t a, int64_t b, cudaStream_t s);
void stencil_box_in(Plan& P, const double* u, int64_t p0, int64_t p1, cudaStream_t s);
void stencil_box_out(Plan& P, const double* u, double* out, int64_t q0, int64_t q1, cudaStream_t s);
int stencil_components(const Plan& P);
int stencil_reach_rows(const Plan& P);   // axis-0 rows an output row reads on either side
int stencil_row_tile(const Plan& P);     // row-range cuts at multiples of it keep results bit-identical
// box FFT mode of method 3 (fft3.cu): 3-D fractional, constant horizon
BoxFft* boxfft_setup(const Plan& P, double alpha);
void boxfft_apply(Plan& P, BoxFft& B, const double* u, const double* scale, double scale0, const double* diag,
                  double* out, cudaStream_t s);
void boxfft_in(Plan& P, BoxFft& B, const double* u, int64_t p0, int64_t p1, cudaStream_t s);
void boxfft_out(Plan& P, BoxFft& B, const double* u, const double* scale, double scale0, const double* diag,
                double* out, int64_t q0, int64_t q1, cudaStream_t s, int parts = 15);
int boxfft_launches(const BoxFft& B);
int boxfft_length(const BoxFft& B);
void boxfft_free(BoxFft* B);

// device BLAS-1 (solve.cu)
size_t dot_scratch_doubles();
void dev_dot(const double* a, const double* b, const double* chk, int64_t n, double* scratch, int* bad,
             cudaStream_t s);   // result at scratch[dot_scratch_doubles() - 1]
void dev_axpy2(double* u, double* r, const double* p, const double* ap, double alpha, int64_t n, cudaStream_t s);
void dev_xpby(double* p, const double* z, double beta, int64_t n, cudaStream_t s);
void dev_negate(double* x, int64_t n, cudaStream_t s);
void dev_diff(double* d, const double* f, const double* x, int64_t n, cudaStream_t s);

// Step-1 tree instruments (tree.cpp), host side
void tree_decompose(int dim, int64_t n, const double* center, double radius, std::vector<int>& levels,
                    std::vector<int64_t>& indices, int64_t& recur_calls);
void tree_count(int dim, int64_t n, const double* radii, int64_t& recur_calls, int64_t& panels);
int64_t tree_moments(int dim, int64_t n, int K, const double* u, double* out);

// host algebra (algebra.cpp)
std::vector<double> match_polynomial(int K, double c);
void match_polynomial_exact(int K, int64_t* num, int64_t* den);
void split_kernel(int K, double c, std::vector<double>& poly, std::vector<double>& tail);
ExpSum fit_exponential_sum(double alpha, int near, int64_t dmax, double tol);
ExpSum fit_exponential_sum_narrow(double alpha, int64_t lo, int64_t hi, double tol, int max_terms);

}  // namespace nlg
