/* oracle/nonloc_oracle.h — restated CPU oracle for the nonlocal-apply hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker. The product (paper_1905_08375_b200/) never links or calls it.
 *
 * Parity status: PINNED. tests/test_oracle_pins.py checks this restatement
 * against (a) the compiled reference (oracle/_ref, built from
 * /root/reference/proj/src by oracle/Makefile) on every case the reference can
 * express, and (b) the committed golden vectors in tests/golden/ generated from
 * the compiled reference by tests/golden/make_golden.py.
 *
 * Everything is plain C11 fp64, compiled with -ffp-contract=off like the
 * reference (/root/reference/proj/CMakeLists.txt:11-12).
 */
#ifndef NONLOC_ORACLE_H
#define NONLOC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_LEAF = 0, ORC_POINT = 1 };            /* InclusionRule, operators.hpp:16 */
enum { ORC_MASS = 0, ORC_DIFFERENCE = 1 };       /* ApplyForm, operators.hpp:20 */
enum { ORC_CLIP = 0, ORC_COLLAR = 1 };           /* exterior: clip (operators.cpp:36-38) or zero collar */

/* Kernel families. The first four follow ProfileFamily (kernel.hpp:43-48) and
 * the reference's omega = C/delta^{d+2} * gamma(r/delta) (kernel.cpp:275-287).
 * FRACTIONAL and PERIDYNAMIC are the BASELINE-only kernels (no reference). */
enum {
  ORC_TRUNCATED = 0,   /* gamma = p(s) = sum_j poly[j] s^{2j}          (kernel.cpp:106-112) */
  ORC_INVERSE_S = 1,   /* gamma = c/s                                  (kernel.cpp:169-171) */
  ORC_CONICAL = 2,     /* gamma = c/s (1-s)                            (kernel.cpp:172-175) */
  ORC_KAPPA = 3,       /* gamma = kappa(s), split remainder            (kernel.cpp:114-126) */
  ORC_FRACTIONAL = 4,  /* omega = C(x) kw(x,y) |y-x|^{-alpha}, Point rule, Difference form */
  ORC_PERIDYNAMIC = 5  /* vector: out = -h^d sum c(x)/|r| (e.(u_y-u_x)) e, Point rule */
};

/* Which reference routine's bookkeeping the loop follows. */
enum {
  ORC_ROUTE_TRUNCATED = 0, /* apply_truncated_dense: self included, front=C/delta^{d+2} (operators.cpp:169-204) */
  ORC_ROUTE_SMOOTH = 1,    /* apply_smooth_dense: skip self, r>=delta skipped (operators.cpp:206-234) */
  ORC_ROUTE_FULL = 2       /* apply_full_dense: skip self, w==0 skipped, window by reach (operators.cpp:236-260) */
};

typedef struct orc_desc {
  int dim;               /* 1..3 */
  int64_t n;             /* nodes per axis; h = 1/n, x_k = (k+1/2) h */
  int family;            /* ORC_TRUNCATED.. */
  int route;             /* ORC_ROUTE_* (ignored for FRACTIONAL / PERIDYNAMIC) */
  const double* poly;    /* TRUNCATED / KAPPA: p(s) coefficients in s^2 */
  int npoly;
  const double* tail;    /* KAPPA: tail(s) coefficients in s (kernel.cpp:121-125) */
  int ntail;
  int order;             /* KAPPA: K, (1-s)^{K+1} factor */
  double c;              /* profile constant (InverseS / Conical / kappa scale) */
  double alpha;          /* FRACTIONAL exponent, omega ~ r^-alpha */
  int rule;              /* ORC_LEAF / ORC_POINT (TRUNCATED route only) */
  int form;              /* ORC_MASS / ORC_DIFFERENCE (TRUNCATED route only) */
  int exterior;          /* ORC_CLIP / ORC_COLLAR (FRACTIONAL, PERIDYNAMIC, FULL) */
  int divergence;        /* horizon(x,y) = (delta_x+delta_y)/2 (kernel.cpp:270-273) */
  const double* delta;   /* per-node delta(x_i), or NULL -> delta0 */
  double delta0;
  double reach;          /* window radius for ROUTE_FULL (HorizonField::max_radius) */
  const double* coeff;   /* per-node C(x_i), or NULL -> coeff0 */
  double coeff0;
  const double* kappa;   /* per-node kappa for (kappa_x+kappa_y)/2 weighting, or NULL */
} orc_desc;

/* Reference bench.cpp:10-16 restated: std::mt19937_64(seed) +
 * uniform_real_distribution<double>(-1,1) as libstdc++ implements it. */
void orc_random_vector(int64_t n, uint64_t seed, double* out);

/* Matching polynomial p^{2K} for c/s (kernel.cpp:26-51,184-207), K <= 6. */
int orc_match_polynomial(int K, double c, double* coeffs);

/* Scalar apply. targets == NULL -> all N nodes (out has N entries); else out[t]
 * is the value at node targets[t]. pairs (optional) counts summed pairs exactly
 * as the reference's pair_count. Returns 0 or a negative error code. */
int orc_apply(const orc_desc* d, const double* u, double* out,
              const int64_t* targets, int64_t ntargets, int64_t* pairs);

/* Peridynamics: u and out are SoA planes [dim][N]. */
int orc_apply_peri(const orc_desc* d, const double* u, double* out,
                   const int64_t* targets, int64_t ntargets, int64_t* pairs);

/* GaussianBump horizon per node (kernel.cpp:255-259). */
void orc_bump_horizon(int dim, int64_t n, double delta0, double* out);

/* Exact Leaf-rule / Point-rule membership, the quadrature contract
 * (geometry.cpp:63-76, operators.cpp:71-78). dk = integer offsets y-x. */
int orc_leaf_in(int dim, int64_t n, const int64_t* kx, const int64_t* ky, double delta);
int orc_point_in(int dim, int64_t n, const int64_t* kx, const int64_t* ky, double delta);

#ifdef __cplusplus
}
#endif
#endif
