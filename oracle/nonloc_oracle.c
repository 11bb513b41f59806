/* oracle/nonloc_oracle.c — restated CPU oracle (plain C11, fp64).
 *
 * TEST INFRASTRUCTURE ONLY (see nonloc_oracle.h). Each routine restates the
 * reference algorithm it cites, in the same floating-point operation order, so
 * that results agree with the compiled reference to rounding (1e-15 relative)
 * and inclusion sets agree exactly. Loops are literal O(N (delta/h)^d) direct
 * sums: this is a checker, not a fast path.
 */
#include "nonloc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- mt19937_64 + libstdc++ uniform_real_distribution (bench.cpp:10-16) ---- */

typedef struct { uint64_t mt[312]; int idx; } mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  static const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

void orc_random_vector(int64_t n, uint64_t seed, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  const double two64 = 18446744073709551616.0;
  for (int64_t i = 0; i < n; ++i) {
    /* generate_canonical<double,53>: one 64-bit draw, (double)x / 2^64, < 1 */
    double r = (double)mt64_next(&g) / two64;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    out[i] = r * (1.0 - -1.0) + -1.0;
  }
}

/* ---- matching polynomial for c/s (kernel.cpp:26-51, 184-207) ---- */

static long long ff(long long n, long long m) {
  long long r = 1;
  for (long long i = 0; i < m; ++i) r *= (n - i);
  return r;
}

static long long gcdll(long long a, long long b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) { long long t = a % b; a = b; b = t; }
  return a;
}

typedef struct { long long p, q; } rat;
static rat rnorm(long long p, long long q) {
  if (q < 0) { p = -p; q = -q; }
  long long g = gcdll(p, q);
  if (g > 1) { p /= g; q /= g; }
  if (p == 0) q = 1;
  rat r = {p, q};
  return r;
}
static rat rsub(rat a, rat b) { return rnorm(a.p * b.q - b.p * a.q, a.q * b.q); }
static rat rmul(rat a, rat b) { return rnorm(a.p * b.p, a.q * b.q); }
static rat rdiv(rat a, rat b) { return rnorm(a.p * b.q, a.q * b.p); }

int orc_match_polynomial(int K, double c, double* coeffs) {
  if (K < 0 || K > 6) return -1;
  const int n = K + 1;
  rat a[7][7], b[7];
  for (int m = 0; m < n; ++m) {
    for (int j = 0; j < n; ++j) a[m][j] = rnorm(2 * j >= m ? ff(2 * j, m) : 0, 1);
    b[m] = rnorm((m % 2 == 0 ? 1 : -1) * ff(m, m), 1);
  }
  for (int col = 0; col < n; ++col) {
    int piv = col;
    while (piv < n && a[piv][col].p == 0) ++piv;
    if (piv == n) return -2;
    for (int j = 0; j < n; ++j) { rat t = a[col][j]; a[col][j] = a[piv][j]; a[piv][j] = t; }
    { rat t = b[col]; b[col] = b[piv]; b[piv] = t; }
    for (int r = 0; r < n; ++r) {
      if (r == col || a[r][col].p == 0) continue;
      rat f = rdiv(a[r][col], a[col][col]);
      for (int cc = col; cc < n; ++cc) a[r][cc] = rsub(a[r][cc], rmul(f, a[col][cc]));
      b[r] = rsub(b[r], rmul(f, b[col]));
    }
  }
  for (int r = 0; r < n; ++r) {
    rat v = rdiv(b[r], a[r][r]);
    coeffs[r] = c * (double)v.p / (double)v.q;
  }
  return 0;
}

/* ---- geometry predicates (geometry.cpp:47-97) ---- */

static double node_coord(int64_t k, double h) { return ((double)k + 0.5) * h; }

/* cube_intersects_ball with the leaf box [k h,(k+1)h]^d (operators.cpp:44-51) */
static int leaf_in(int dim, const int64_t* ky, const double* x, double h, double r) {
  double dmin = 0.0;
  for (int j = 0; j < dim; ++j) {
    const double lo = (double)ky[j] * h, hi = (double)(ky[j] + 1) * h;
    if (lo > x[j]) { const double d = lo - x[j]; dmin += d * d; }
    else if (hi < x[j]) { const double d = hi - x[j]; dmin += d * d; }
  }
  return dmin < r * r;
}

/* dist (operators.cpp:71-78) */
static double dist(int dim, const double* x, const double* y) {
  double r2 = 0.0;
  for (int j = 0; j < dim; ++j) { const double d = y[j] - x[j]; r2 += d * d; }
  return sqrt(r2);
}

int orc_leaf_in(int dim, int64_t n, const int64_t* kx, const int64_t* ky, double delta) {
  const double h = 1.0 / (double)n;
  double x[3];
  for (int j = 0; j < dim; ++j) x[j] = node_coord(kx[j], h);
  return leaf_in(dim, ky, x, h, delta);
}

int orc_point_in(int dim, int64_t n, const int64_t* kx, const int64_t* ky, double delta) {
  const double h = 1.0 / (double)n;
  double x[3], y[3];
  for (int j = 0; j < dim; ++j) { x[j] = node_coord(kx[j], h); y[j] = node_coord(ky[j], h); }
  return dist(dim, x, y) < delta;
}

/* ---- helpers (operators.cpp:20-100) ---- */

static double delta_power(int dim, double delta) {
  double p = delta * delta;
  for (int j = 0; j < dim; ++j) p *= delta;
  return p;
}

static double hd_weight(int dim, double h) {
  double w = h;
  for (int j = 1; j < dim; ++j) w *= h;
  return w;
}

static double ball_volume(int dim, double r) {
  const double pi = 3.141592653589793238462643383279502884; /* std::numbers::pi */
  switch (dim) {
    case 1: return 2.0 * r;
    case 2: return pi * r * r;
    default: return 4.0 / 3.0 * pi * r * r * r;
  }
}

/* MatchedPolynomial::operator() — Horner in s^2 (kernel.cpp:106-112) */
static double poly_eval(const double* cf, int np, double s) {
  const double t = s * s;
  double acc = 0.0;
  for (int j = np - 1; j >= 0; --j) acc = acc * t + cf[j];
  return acc;
}

/* SplitKernel::kappa (kernel.cpp:114-126) */
static double kappa_eval(const orc_desc* d, double s) {
  s = fabs(s);
  if (s >= 1.0) return 0.0;
  if (s < 0.5) return d->c / s - poly_eval(d->poly, d->npoly, s);
  const double u = 1.0 - s;
  double f = 1.0;
  for (int i = 0; i <= d->order; ++i) f *= u;
  double acc = 0.0;
  for (int j = d->ntail - 1; j >= 0; --j) acc = acc * s + d->tail[j];
  return f * acc / s;
}

/* eval_profile (kernel.cpp:164-182) */
static double profile_eval(const orc_desc* d, double s) {
  s = fabs(s);
  if (s >= 1.0) return 0.0;
  switch (d->family) {
    case ORC_INVERSE_S: return d->c / s;
    case ORC_CONICAL: return d->c / s * (1.0 - s);
    case ORC_KAPPA: return kappa_eval(d, s);
    case ORC_TRUNCATED: return poly_eval(d->poly, d->npoly, s);
    default: return 0.0;
  }
}

static void multi_index(int dim, int64_t n, int64_t flat, int64_t* k) {
  for (int j = dim - 1; j >= 0; --j) { k[j] = flat % n; flat /= n; }
}

typedef struct { int64_t lo[3], hi[3]; } win;

/* window_around (operators.cpp:31-42); clip=0 keeps exterior indices (collar). */
static win window_around(int dim, int64_t n, double h, const double* x, double radius, int clip) {
  win w;
  for (int j = 0; j < 3; ++j) { w.lo[j] = 0; w.hi[j] = 0; }
  for (int j = 0; j < dim; ++j) {
    const double lo = (x[j] - radius) / h - 1.0;
    const double hi = (x[j] + radius) / h + 1.0;
    int64_t l = (int64_t)floor(lo), u = (int64_t)ceil(hi);
    if (clip) { if (l < 0) l = 0; if (u > n - 1) u = n - 1; }
    w.lo[j] = l;
    w.hi[j] = u;
  }
  return w;
}

static double field(const double* a, double a0, int64_t i) { return a ? a[i] : a0; }

static int inside(int dim, int64_t n, const int64_t* k) {
  for (int j = 0; j < dim; ++j) if (k[j] < 0 || k[j] >= n) return 0;
  return 1;
}

static int64_t flatten(int dim, int64_t n, const int64_t* k) {
  int64_t f = 0;
  for (int j = 0; j < dim; ++j) f = f * n + k[j];
  return f;
}

/* One target of the scalar operator. */
static double apply_one(const orc_desc* d, const double* u, int64_t i, int64_t* pairs) {
  const int dim = d->dim;
  const int64_t n = d->n;
  const double h = 1.0 / (double)n;
  const double hd = hd_weight(dim, h);
  int64_t ki[3] = {0, 0, 0};
  multi_index(dim, n, i, ki);
  double x[3] = {0, 0, 0};
  for (int j = 0; j < dim; ++j) x[j] = node_coord(ki[j], h);
  const double delta = field(d->delta, d->delta0, i);
  const double ui = u[i];
  const double ci = field(d->coeff, d->coeff0, i);
  const int collar = d->exterior == ORC_COLLAR;

  if (d->family == ORC_FRACTIONAL) {
    /* BASELINE operator, Point rule, Difference form; clip or zero collar. */
    const win w = window_around(dim, n, h, x, delta, !collar);
    const double ki_kappa = d->kappa ? d->kappa[i] : 1.0;
    double acc = 0.0;
    int64_t k[3] = {0, 0, 0};
    for (k[0] = w.lo[0]; k[0] <= w.hi[0]; ++k[0])
      for (k[1] = w.lo[1]; k[1] <= w.hi[1]; ++k[1])
        for (k[2] = w.lo[2]; k[2] <= w.hi[2]; ++k[2]) {
          double y[3] = {0, 0, 0};
          for (int j = 0; j < dim; ++j) y[j] = node_coord(k[j], h);
          const int in_dom = inside(dim, n, k);
          const int64_t f = in_dom ? flatten(dim, n, k) : -1;
          if (f == i) continue;
          const double r = dist(dim, x, y);
          if (!(r < delta)) continue;
          double c = ci;
          if (d->kappa) c *= 0.5 * (ki_kappa + (in_dom ? d->kappa[f] : ki_kappa));
          const double wgt = c * pow(r, -d->alpha);
          const double uk = in_dom ? u[f] : 0.0;
          acc += wgt * (uk - ui);
          if (pairs) ++*pairs;
        }
    return hd * acc;
  }

  if (d->route == ORC_ROUTE_TRUNCATED) {
    /* apply_truncated_dense (operators.cpp:169-204) */
    const win w = window_around(dim, n, h, x, delta, 1);
    double acc = 0.0;
    int64_t k[3] = {0, 0, 0};
    for (k[0] = w.lo[0]; k[0] <= w.hi[0]; ++k[0])
      for (k[1] = w.lo[1]; k[1] <= w.hi[1]; ++k[1])
        for (k[2] = w.lo[2]; k[2] <= w.hi[2]; ++k[2]) {
          double y[3] = {0, 0, 0};
          for (int j = 0; j < dim; ++j) y[j] = node_coord(k[j], h);
          const int in = d->rule == ORC_POINT ? dist(dim, x, y) < delta
                                              : leaf_in(dim, k, x, h, delta);
          if (!in) continue;
          if (pairs) ++*pairs;
          const int64_t f = flatten(dim, n, k);
          const double v = poly_eval(d->poly, d->npoly, dist(dim, x, y) / delta);
          acc += d->form == ORC_MASS ? v * u[f] : v * (u[f] - ui);
        }
    const double front = ci / delta_power(dim, delta);
    return d->form == ORC_MASS ? front * (hd * acc - ball_volume(dim, delta) * ui)
                               : front * hd * acc;
  }

  if (d->route == ORC_ROUTE_SMOOTH) {
    /* apply_smooth_dense (operators.cpp:206-234) */
    const win w = window_around(dim, n, h, x, delta, 1);
    const double front = 1.0 / delta_power(dim, delta);
    double acc = 0.0;
    int64_t k[3] = {0, 0, 0};
    for (k[0] = w.lo[0]; k[0] <= w.hi[0]; ++k[0])
      for (k[1] = w.lo[1]; k[1] <= w.hi[1]; ++k[1])
        for (k[2] = w.lo[2]; k[2] <= w.hi[2]; ++k[2]) {
          const int64_t f = flatten(dim, n, k);
          if (f == i) continue;
          double y[3] = {0, 0, 0};
          for (int j = 0; j < dim; ++j) y[j] = node_coord(k[j], h);
          const double r = dist(dim, x, y);
          if (r >= delta) continue;
          if (pairs) ++*pairs;
          acc += ci * front * kappa_eval(d, r / delta) * (u[f] - ui);
        }
    return hd * acc;
  }

  /* ROUTE_FULL: apply_full_dense with eval_omega (operators.cpp:236-260,
   * kernel.cpp:275-287); optional zero collar. */
  {
    const double reach = d->reach > 0.0 ? d->reach : delta;
    const win w = window_around(dim, n, h, x, reach, !collar);
    double acc = 0.0;
    int64_t k[3] = {0, 0, 0};
    for (k[0] = w.lo[0]; k[0] <= w.hi[0]; ++k[0])
      for (k[1] = w.lo[1]; k[1] <= w.hi[1]; ++k[1])
        for (k[2] = w.lo[2]; k[2] <= w.hi[2]; ++k[2]) {
          const int in_dom = inside(dim, n, k);
          const int64_t f = in_dom ? flatten(dim, n, k) : -1;
          if (f == i) continue;
          double y[3] = {0, 0, 0};
          for (int j = 0; j < dim; ++j) y[j] = node_coord(k[j], h);
          const double r = dist(dim, x, y);
          double dl = delta;
          if (d->divergence) dl = 0.5 * (delta + (in_dom ? field(d->delta, d->delta0, f) : delta));
          if (r >= dl) continue;
          double c = ci;
          if (d->kappa) c *= 0.5 * (d->kappa[i] + (in_dom ? d->kappa[f] : d->kappa[i]));
          const double wgt = c / delta_power(dim, dl) * profile_eval(d, r / dl);
          if (wgt == 0.0) continue;
          if (pairs) ++*pairs;
          acc += wgt * ((in_dom ? u[f] : 0.0) - ui);
        }
    return hd * acc;
  }
}

int orc_apply(const orc_desc* d, const double* u, double* out,
              const int64_t* targets, int64_t ntargets, int64_t* pairs) {
  if (!d || d->dim < 1 || d->dim > 3 || d->n < 1) return -1;
  int64_t N = 1;
  for (int j = 0; j < d->dim; ++j) N *= d->n;
  const int64_t cnt = targets ? ntargets : N;
  for (int64_t t = 0; t < cnt; ++t) {
    const int64_t i = targets ? targets[t] : t;
    if (i < 0 || i >= N) return -2;
    out[t] = apply_one(d, u, i, pairs);
  }
  return 0;
}

/* Linear bond-based peridynamics (BASELINE cfg3; no reference):
 *   out(x) = -h^d sum_{y != x, |y-x| < delta(x)} c(x)/|y-x| (e.(u_y-u_x)) e,
 *   e = (y-x)/|y-x|; u, out SoA [dim][N]; exterior: clip or zero collar. */
int orc_apply_peri(const orc_desc* d, const double* u, double* out,
                   const int64_t* targets, int64_t ntargets, int64_t* pairs) {
  if (!d || d->dim < 1 || d->dim > 3) return -1;
  const int dim = d->dim;
  const int64_t n = d->n;
  int64_t N = 1;
  for (int j = 0; j < dim; ++j) N *= n;
  const double h = 1.0 / (double)n;
  const double hd = hd_weight(dim, h);
  const int collar = d->exterior == ORC_COLLAR;
  const int64_t cnt = targets ? ntargets : N;
  for (int64_t t = 0; t < cnt; ++t) {
    const int64_t i = targets ? targets[t] : t;
    if (i < 0 || i >= N) return -2;
    int64_t ki[3] = {0, 0, 0};
    multi_index(dim, n, i, ki);
    double x[3] = {0, 0, 0};
    for (int j = 0; j < dim; ++j) x[j] = node_coord(ki[j], h);
    const double delta = field(d->delta, d->delta0, i);
    const double ci = field(d->coeff, d->coeff0, i);
    const win w = window_around(dim, n, h, x, delta, !collar);
    double acc[3] = {0, 0, 0};
    int64_t k[3] = {0, 0, 0};
    for (k[0] = w.lo[0]; k[0] <= w.hi[0]; ++k[0])
      for (k[1] = w.lo[1]; k[1] <= w.hi[1]; ++k[1])
        for (k[2] = w.lo[2]; k[2] <= w.hi[2]; ++k[2]) {
          const int in_dom = inside(dim, n, k);
          const int64_t f = in_dom ? flatten(dim, n, k) : -1;
          if (f == i) continue;
          double y[3] = {0, 0, 0};
          for (int j = 0; j < dim; ++j) y[j] = node_coord(k[j], h);
          const double r = dist(dim, x, y);
          if (!(r < delta)) continue;
          if (pairs) ++*pairs;
          double proj = 0.0;
          double e[3] = {0, 0, 0};
          for (int j = 0; j < dim; ++j) {
            e[j] = (y[j] - x[j]) / r;
            const double du = (in_dom ? u[(int64_t)j * N + f] : 0.0) - u[(int64_t)j * N + i];
            proj += e[j] * du;
          }
          const double wgt = ci / r;
          for (int j = 0; j < dim; ++j) acc[j] += wgt * proj * e[j];
        }
    for (int j = 0; j < dim; ++j) out[(int64_t)j * cnt + t] = -hd * acc[j];
  }
  return 0;
}

/* HorizonField::operator() for GaussianBump (kernel.cpp:255-259), per node,
 * with the same libm exp the reference calls. */
void orc_bump_horizon(int dim, int64_t n, double delta0, double* out) {
  const double h = 1.0 / (double)n;
  int64_t N = 1;
  for (int j = 0; j < dim; ++j) N *= n;
  int64_t stride = N / n; /* axis 0 is slowest */
  for (int64_t i = 0; i < N; ++i) {
    const double x0 = node_coord(i / stride, h);
    const double dd = x0 - 0.5;
    out[i] = delta0 * (1.0 + exp(-20.0 * dd * dd));
  }
}
