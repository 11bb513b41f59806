/* include/nlgpu.h — C-ABI of the B200-native nonlocal-apply hot path.
 *
 * This is the drop-in boundary. Plain C types, plain
 * pointers and sizes; no torch, no C++ types. A plan owns its device buffers;
 * host-pointer entry points do the H2D/D2H copies themselves (blocking), the
 * *_dev entry points take device pointers and a cudaStream_t (as void*) and
 * are asynchronous on that stream (Krylov-resident use).
 *
 * Reference interfaces each entry point replaces (/root/reference/proj/...):
 *   nlg_plan_create      TruncatedOperator::TruncatedOperator  include/nonloc/operators.hpp:32
 *                        (Step 1: caches delta_, coeff_  src/operators.cpp:102-124), and the
 *                        KernelSpec/Grid setup of apply_*_dense  operators.hpp:58-75
 *   nlg_apply_fast       TruncatedOperator::apply               operators.hpp:34, operators.cpp:126-167
 *                        (and, for the BASELINE kernels, the fast apply the reference lacks)
 *   nlg_apply_direct     apply_truncated_dense                  operators.hpp:58-62, operators.cpp:169-204
 *                        apply_smooth_dense                     operators.hpp:66-70, operators.cpp:206-234
 *                        apply_full_dense                       operators.hpp:73-75, operators.cpp:236-260
 *   nlg_counters         TruncatedOperator::{step2,step3}_ops / pair_count out-params
 *                        operators.hpp:39-42, operators.cpp:193,225,253
 *   nlg_match_polynomial match_polynomial                       kernel.hpp:63-64, kernel.cpp:184-207
 *   nlg_split            split                                  kernel.hpp:66, kernel.cpp:209-245
 *   nlg_last_error       the what() text of the reference's exceptions
 *                        (std::invalid_argument / domain_error / out_of_range / runtime_error)
 */
#ifndef NLGPU_H
#define NLGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NLG_ABI_VERSION 1

typedef struct nlg_plan nlg_plan;

/* Status codes; the C++ shim rethrows them as the reference's exception types
 * (include/nonloc/*.hpp, SURVEY §8(b) "Errors"). */
typedef enum {
  NLG_OK = 0,
  NLG_EINVAL = 1,      /* std::invalid_argument (config / size errors)       */
  NLG_EDOMAIN = 2,     /* std::domain_error (singular evaluation at s = 0)   */
  NLG_ERANGE = 3,      /* std::out_of_range (bad node index)                 */
  NLG_ERUNTIME = 4,    /* std::runtime_error                                 */
  NLG_ECUDA = 5,       /* CUDA error            -> std::runtime_error        */
  NLG_ENCCL = 6,       /* collective error      -> std::runtime_error        */
  NLG_EUNSUPPORTED = 7 /* valid request this build does not implement -> invalid_argument */
} nlg_status;

enum { NLG_LEAF = 0, NLG_POINT = 1 };            /* InclusionRule (operators.hpp:16) */
enum { NLG_MASS = 0, NLG_DIFFERENCE = 1 };       /* ApplyForm (operators.hpp:20)     */
enum { NLG_CLIP = 0, NLG_COLLAR = 1 };           /* exterior: clipped window (operators.cpp:36-38)
                                                    or zero volume-constraint collar */
enum {
  NLG_TRUNCATED = 0,   /* gamma(s) = p(s), even polynomial in s (kernel.cpp:106-112)      */
  NLG_INVERSE_S = 1,   /* gamma(s) = c/s                                                   */
  NLG_CONICAL = 2,     /* gamma(s) = c/s (1-s)                                             */
  NLG_KAPPA = 3,       /* gamma(s) = kappa(s), the split remainder (kernel.cpp:114-126)    */
  NLG_FRACTIONAL = 4,  /* omega(x,y) = C(x) kw(x,y) |y-x|^-alpha (BASELINE cfg0/1/2/4)    */
  NLG_PERIDYNAMIC = 5  /* vector: -h^d sum C(x)/|y-x| (e.(u_y-u_x)) e (BASELINE cfg3)      */
};
/* Which reference routine's bookkeeping a direct apply follows. */
enum {
  NLG_ROUTE_TRUNCATED = 0, /* apply_truncated_dense: self included, Mass/Difference, Leaf/Point */
  NLG_ROUTE_SMOOTH = 1,    /* apply_smooth_dense:   self skipped, Point, Difference            */
  NLG_ROUTE_FULL = 2       /* apply_full_dense:     self skipped, Point, Difference, eval_omega */
};

/* Operator description. Mirrors KernelSpec + Grid (kernel.hpp:97-108,
 * geometry.hpp:18-26) flattened to POD: x-dependent parts arrive as host
 * arrays evaluated at the nodes (delta_ / coeff_ of operators.cpp:119-120).
 * Arrays are row-major (axis 0 slowest, geometry.cpp:86-97) over the plan's
 * INPUT rows (see row_begin / row_end), or NULL for the scalar value. */
typedef struct nlg_desc {
  int dim;               /* 1, 2 or 3                                          */
  int64_t n;             /* nodes per axis, h = 1/n, x_k = (k+1/2)h            */
  int family;            /* NLG_TRUNCATED .. NLG_PERIDYNAMIC                   */
  int route;             /* NLG_ROUTE_* (profile families only)                */
  const double* poly;    /* TRUNCATED / KAPPA: p(s) = sum_j poly[j] s^{2j}     */
  int npoly;
  const double* tail;    /* KAPPA: tail(s) = sum_j tail[j] s^j                 */
  int ntail;
  int order;             /* KAPPA: K of the (1-s)^{K+1} factor                 */
  double c;              /* profile constant                                   */
  double alpha;          /* FRACTIONAL exponent (d + 2s)                       */
  int rule;              /* NLG_LEAF / NLG_POINT                               */
  int form;              /* NLG_MASS / NLG_DIFFERENCE                          */
  int exterior;          /* NLG_CLIP / NLG_COLLAR                              */
  int divergence;        /* horizon(x,y) = (delta(x)+delta(y))/2 (kernel.cpp:270-273) */
  const double* delta;   /* delta(x_i) per node, or NULL -> delta0             */
  double delta0;
  double reach;          /* window radius (HorizonField::max_radius); <=0: max delta */
  const double* coeff;   /* C(x_i) per node, or NULL -> coeff0                 */
  double coeff0;
  const double* kappa;   /* kappa(x_i) for (kappa(x)+kappa(y))/2 weighting, or NULL */
  /* Slab sharding along axis 0. The plan produces output rows
   * [row_begin, row_end) of axis 0; all per-node arrays above and the u passed
   * to apply cover the INPUT rows [row_begin - halo_lo, row_end + halo_hi),
   * where halo_lo/halo_hi come from nlg_plan_info(). row_end = 0 means the
   * whole grid (no sharding). Per-node arrays must then cover the input rows,
   * so call nlg_halo_rows() first to size them. */
  int64_t row_begin;
  int64_t row_end;
  int device;            /* CUDA device ordinal                                */
} nlg_desc;

typedef struct nlg_info {
  int64_t halo_lo, halo_hi;  /* input rows below / above the output slab       */
  int64_t n_in, n_out;       /* nodes in the input / output slab               */
  int fast_method;           /* 0 direct quadrature, 1 span prefix sums
                                (polynomial kernels), 2 exponential-sum scans
                                (1-D fractional), 3 offset-table stencil
                                (2-D/3-D fractional, 2-D peridynamics),
                                4 centred moment scans (1-D polynomial K = 1..3,
                                Mass form: the reference's Steps 2 + 3)        */
  int exp_terms;             /* far-field terms of the 1-D exponential sum     */
  int near_cells;            /* near-field radius (cells) of the 1-D scan path */
  double far_rel_err;        /* fitted kernel error of the exponential sum     */
  int64_t fft_len;           /* FFT convolution length L: the 1-D far window
                                (method 2) or the x / y box axis of the 3-D
                                constant-horizon mode (method 3); 0 = none     */
  int fft_rows;              /* four-step split L = N1 x fft_rows (fft.cu);
                                0: the cuFFT path for lengths it does not cover */
} nlg_info;

/* Halo rows a slab [row_begin,row_end) needs for this operator, before the
 * per-node arrays exist (uses delta0 / reach / the max of delta). */
nlg_status nlg_halo_rows(const nlg_desc* desc, double delta_max, int64_t* halo);

nlg_status nlg_plan_create(const nlg_desc* desc, nlg_plan** out);
void nlg_plan_destroy(nlg_plan* plan);
nlg_status nlg_plan_info(const nlg_plan* plan, nlg_info* info);

/* Host pointers, blocking. u covers the input rows (components planes
 * [dim][n_in] for PERIDYNAMIC); out covers the output rows. For 2-D / 3-D
 * scalar stencil and box-FFT plans of >= 4 Mi nodes nlg_apply_fast is a
 * chunked pipeline (H2D of input rows, the apply of every output row range
 * whose window is resident, D2H of finished rows, on three streams); pinned
 * host buffers let the copies overlap. NLG_NO_PIPELINE=1 disables it. */
nlg_status nlg_apply_fast(nlg_plan* plan, const double* u, double* out);
nlg_status nlg_apply_direct(nlg_plan* plan, const double* u, double* out, int64_t* pair_count);

/* Device pointers, asynchronous on `stream` (cudaStream_t, may be NULL). */
nlg_status nlg_apply_fast_dev(nlg_plan* plan, const double* u_dev, double* out_dev, void* stream);
nlg_status nlg_apply_direct_dev(nlg_plan* plan, const double* u_dev, double* out_dev,
                                int64_t* pair_count_dev, void* stream);

/* Split-phase device apply for sharded plans (multi-GPU halo overlap):
 * _begin enqueues the part of the fast apply that does not read u's halo rows
 * (box FFT mode: the x / y transforms of the owned planes; 2-D / 3-D scalar
 * stencil slabs: the output rows whose window lies in the owned input rows),
 * _end the rest once
 * the halo rows of u_dev hold the neighbours' values. begin + end ==
 * nlg_apply_fast_dev; for methods without a halo-independent part _begin does
 * nothing. Same stream for both calls. */
nlg_status nlg_apply_fast_dev_begin(nlg_plan* plan, const double* u_dev, double* out_dev, void* stream);
nlg_status nlg_apply_fast_dev_end(nlg_plan* plan, const double* u_dev, double* out_dev, void* stream);

/* Direct apply at a subset of output nodes (flat indices into the output
 * slab); used for sampled parity at BASELINE sizes. Host pointers, blocking.
 * pair_count (optional) receives the pairs summed over those targets, counted
 * as the reference's pair_count (operators.cpp:193,225,253). */
nlg_status nlg_apply_direct_at(nlg_plan* plan, const double* u, const int64_t* targets,
                               int64_t ntargets, double* out, int64_t* pair_count);

/* Counters in the reference's semantics: pairs summed by the last direct apply
 * (operators.cpp:193,225,253); number of fast applies issued. */
nlg_status nlg_counters(const nlg_plan* plan, int64_t* pairs, int64_t* fast_applies);

/* Per-stage CUDA-event timing of this plan's kernels (off by default).
 * Stages: 0 direct, 1 span scan, 2 span eval, 3 exp-sum aggregate, 4 exp-sum
 * carry, 5 exp-sum main, 6 near+combine, 7 stencil, 8 exp-sum FFT (cuFFT
 * chain), 9 box FFT (unused), 10 box tie band, 11-15 box FFT passes PA..PE,
 * 16-18 four-step FFT passes P1..P3. With profiling on, side streams are
 * folded into the apply's stream so stage times never overlap (one kernel per
 * stage except 4, 7 and 8). nlg_stage_times returns (and resets) the
 * accumulated milliseconds and launch counts per stage: the caller's arrays
 * hold NLG_NUM_STAGES slots. */
#define NLG_NUM_STAGES 19
nlg_status nlg_set_profiling(nlg_plan* plan, int on);
nlg_status nlg_stage_times(nlg_plan* plan, double* ms, int64_t* launches, int* nstages);
/* Total kernels this plan has launched. */
nlg_status nlg_launch_count(const nlg_plan* plan, int64_t* launches);

/* Kernel algebra (host setup, exact rationals for K <= 4 like kernel.cpp:26-51). */
nlg_status nlg_match_polynomial(int K, double c, double* coeffs /* K+1 */);
nlg_status nlg_match_polynomial_exact(int K, int64_t* num, int64_t* den);   /* c = 1, K <= 6 */
nlg_status nlg_split(int K, double c, double* poly /* K+1 */, double* tail /* >= K+1 */,
                     int* ntail);

/* Far-field exponential sum used by the 1-D fast path (host, for tests and
 * diagnostics): d^-alpha ~= sum_m weight[m] exp(-rate[m] d) on d in
 * [near+1, dmax]. rate/weight must hold 64 entries; *rel_err is the max
 * relative error over every integer d in the window. */
nlg_status nlg_expsum_fit(double alpha, int near, int64_t dmax, double* rate, double* weight,
                          int* terms, double* rel_err);

/* Matrix view of the direct operators (routes 0-2 and FRACTIONAL; not
 * PERIDYNAMIC): out = A^T v for the plan's operator A (apply_direct = A u).
 * The transpose is what CGNR needs for non-symmetric operators (variable
 * horizons, coefficient_fn); the reference assembles the dense matrix for
 * this (tools/nonloc_main.cpp:200-219). Host / device pointers as above. */
nlg_status nlg_apply_transpose(nlg_plan* plan, const double* v, double* out);
nlg_status nlg_apply_transpose_dev(nlg_plan* plan, const double* v_dev, double* out_dev, void* stream);

/* Dense row-major N x N matrix of an unsharded plan's direct operator
 * (reference assemble_dense_matrix, operators.cpp:262-303). a: host, N^2. */
nlg_status nlg_assemble_dense(nlg_plan* plan, double* a_rowmajor);

/* Matrix-free Krylov solve of A u = f with A = -L (the negated operator, the
 * reference's solve_dirichlet convention, src/solve.cpp:32-108), vectors
 * resident on the device: CG, or CGNR on the normal equations with the GPU
 * transpose. L is the plan's fast apply (or its direct apply with
 * NLG_SOLVE_DIRECT). Unsharded scalar plans only. Non-convergence is reported,
 * a non-finite operator value is NLG_ERUNTIME (check_finite, solve.cpp:24-28).
 * f, u: host, N doubles. */
#define NLG_SOLVE_CG 0
#define NLG_SOLVE_CGNR 1
#define NLG_SOLVE_DIRECT 0x10
typedef struct {
  int method;              /* NLG_SOLVE_CG or NLG_SOLVE_CGNR                  */
  int converged;           /* final_residual <= tol                            */
  int64_t iterations;
  double final_residual;   /* ||f - A u||_2 / ||f||_2, recomputed at the end   */
} nlg_solve_report;
nlg_status nlg_solve_dirichlet(nlg_plan* plan, const double* f, double tol, int64_t max_iter, int method,
                               double* u, nlg_solve_report* report);

/* Short exponential sum for |d|^-alpha on the narrow window [lo, hi]
 * (far-end tails of the 1-D fractional fast path); arrays of max_terms. */
nlg_status nlg_expsum_fit_narrow(double alpha, int64_t lo, int64_t hi, double tol, int max_terms, double* rate,
                                 double* weight, int* terms, double* rel_err);

/* Step-1 tree instruments of the reference (tree.hpp:31-53), host side: the
 * panels of decompose_region for one ball (pre-order, up to `cap` written;
 * npanels = full count), the recursion-call and panel totals over every node
 * of an n^dim grid with per-node radii (count_recur_calls; the panel total
 * times the moment count is the reference's step3_ops per apply), and
 * accumulate_moments (levels 0..L flattened level-major; adds = step2_ops). */
nlg_status nlg_tree_decompose(int dim, int64_t n, const double* center, double radius, int64_t cap, int* levels,
                              int64_t* indices, int64_t* npanels, int64_t* recur_calls);
nlg_status nlg_tree_count(int dim, int64_t n, const double* radii, int64_t* recur_calls, int64_t* panels);
nlg_status nlg_tree_moments(int dim, int64_t n, int K, const double* u, double* out, int64_t* adds);

/* Multi-GPU plans: one process, ndev devices. The grid's
 * axis-0 rows are split into ndev slabs (even split), one sharded plan per
 * device; u's halo rows (the reference's window, operators.cpp:31-42) move
 * between neighbouring devices by NCCL point-to-point (ncclCommInitAll over
 * the device list; NCCL loaded at run time, errors and
 * ncclCommGetAsyncError -> NLG_ENCCL), overlapped with the halo-independent
 * part of each slab's apply. A device ordinal repeated in the list (several
 * slabs on one GPU: tests) uses peer copies instead of NCCL.
 * desc covers the WHOLE grid (row_begin = row_end = 0; per-node arrays of
 * n^dim entries); desc->device is ignored. */
typedef struct nlg_group nlg_group;
nlg_status nlg_group_create(const nlg_desc* desc, int ndev, const int* devices, nlg_group** out);
void nlg_group_destroy(nlg_group* group);
/* ndev, whether NCCL carries the halos, and per device: owned rows
 * [row_begin, row_end) and input nodes n_in (arrays of ndev, may be NULL). */
nlg_status nlg_group_info(const nlg_group* group, int* ndev, int* nccl, int64_t* row_begin, int64_t* row_end,
                          int64_t* n_in);
/* Host pointers over the whole grid (components planes [dim][N] for
 * PERIDYNAMIC): owned rows H2D per device, halo exchange device to device,
 * apply, owned output rows D2H. Blocking. */
nlg_status nlg_group_apply_fast(nlg_group* group, const double* u, double* out);
/* Device pointers: u_dev[k] holds device k's input rows (n_in nodes per
 * component; only the owned rows need to be filled, the halos are exchanged
 * inside), out_dev[k] its output rows. Blocking. */
nlg_status nlg_group_apply_fast_dev(nlg_group* group, double* const* u_dev, double* const* out_dev);
/* Text of the last group error on this thread. */
const char* nlg_group_last_error(void);

/* Thread-local text of the last error; "" if none. */
const char* nlg_last_error(void);
int nlg_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NLGPU_H */
