// paper_1905_08375_b200/csrc/algebra.cpp — host-side kernel algebra (plan setup).
//
// match_polynomial: the even polynomial p(s) = sum_j c_j s^{2j} with
//   p^(m)(1) = gamma^(m)(1), m = 0..K, for gamma = c/s (kernel.cpp:26-51, 184-207):
//   sum_j ff(2j, m) c_j = c (-1)^m m!. Solved in exact rationals for K <= 4 (the
//   correctly rounded quotients the reference produces) and by a full-pivot fp64
//   solve above that, as the reference does.
// split_kernel: kappa(s) = c/s - p(s) written as c (1-s)^{K+1} tail(s) / s
//   (kernel.cpp:209-245): tail = (1 - s p1(s)) / (1-s)^{K+1}, exact division.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "plan.hpp"

namespace nlg {

namespace {

using i128 = __int128;

i128 gcd128(i128 a, i128 b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b != 0) {
    i128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}

struct Q {
  i128 p = 0, q = 1;
  Q() = default;
  Q(i128 a, i128 b = 1) : p(a), q(b) {
    if (q < 0) { p = -p; q = -q; }
    i128 g = gcd128(p, q);
    if (g > 1) { p /= g; q /= g; }
    if (p == 0) q = 1;
  }
};
Q operator+(Q a, Q b) { return Q(a.p * b.q + b.p * a.q, a.q * b.q); }
Q operator-(Q a, Q b) { return Q(a.p * b.q - b.p * a.q, a.q * b.q); }
Q operator*(Q a, Q b) { return Q(a.p * b.p, a.q * b.q); }
Q operator/(Q a, Q b) { return Q(a.p * b.q, a.q * b.p); }

long long falling(long long n, long long m) {
  long long r = 1;
  for (long long i = 0; i < m; ++i) r *= (n - i);
  return r;
}

std::vector<Q> matching_exact(int K) {
  const int n = K + 1;
  std::vector<std::vector<Q>> a(n, std::vector<Q>(n));
  std::vector<Q> b(n);
  for (int m = 0; m < n; ++m) {
    for (int j = 0; j < n; ++j) a[m][j] = Q(2 * j >= m ? falling(2 * j, m) : 0);
    b[m] = Q((m % 2 == 0 ? 1 : -1) * falling(m, m));
  }
  for (int col = 0; col < n; ++col) {
    int piv = col;
    while (piv < n && a[piv][col].p == 0) ++piv;
    if (piv == n) throw Error{NLG_ERUNTIME, "singular matching system"};
    std::swap(a[col], a[piv]);
    std::swap(b[col], b[piv]);
    for (int r = 0; r < n; ++r) {
      if (r == col || a[r][col].p == 0) continue;
      const Q f = a[r][col] / a[col][col];
      for (int c = col; c < n; ++c) a[r][c] = a[r][c] - f * a[col][c];
      b[r] = b[r] - f * b[col];
    }
  }
  std::vector<Q> out(n);
  for (int r = 0; r < n; ++r) out[r] = b[r] / a[r][r];
  return out;
}

// K > 4: the matching system in fp64 with complete pivoting (the reference
// switches to a double full-pivot LU there, kernel.cpp:53-70,203-205). The
// largest remaining entry is the pivot at every step; a zero pivot is the
// reference's "singular matching system".
std::vector<double> matching_double(int K, double c) {
  const int n = K + 1;
  if (K > 12) throw Error{NLG_EUNSUPPORTED, "matching order > 12 overflows the system's factorials"};
  std::vector<std::vector<double>> a(n, std::vector<double>(n));
  std::vector<double> b(n);
  for (int m = 0; m < n; ++m) {
    for (int j = 0; j < n; ++j) a[m][j] = 2 * j >= m ? static_cast<double>(falling(2 * j, m)) : 0.0;
    b[m] = c * (m % 2 == 0 ? 1.0 : -1.0) * static_cast<double>(falling(m, m));
  }
  std::vector<int> colperm(n);
  for (int j = 0; j < n; ++j) colperm[j] = j;
  for (int k = 0; k < n; ++k) {
    int pr = k, pc = k;
    double best = 0.0;
    for (int r = k; r < n; ++r)
      for (int q = k; q < n; ++q)
        if (std::fabs(a[r][q]) > best) { best = std::fabs(a[r][q]); pr = r; pc = q; }
    if (best == 0.0) throw Error{NLG_ERUNTIME, "singular matching system"};
    std::swap(a[k], a[pr]);
    std::swap(b[k], b[pr]);
    if (pc != k) {
      for (int r = 0; r < n; ++r) std::swap(a[r][k], a[r][pc]);
      std::swap(colperm[k], colperm[pc]);
    }
    for (int r = k + 1; r < n; ++r) {
      const double f = a[r][k] / a[k][k];
      if (f == 0.0) continue;
      for (int q = k; q < n; ++q) a[r][q] -= f * a[k][q];
      b[r] -= f * b[k];
    }
  }
  std::vector<double> y(n), x(n);
  for (int r = n - 1; r >= 0; --r) {
    double acc = b[r];
    for (int q = r + 1; q < n; ++q) acc -= a[r][q] * y[q];
    y[r] = acc / a[r][r];
  }
  for (int j = 0; j < n; ++j) x[colperm[j]] = y[j];
  return x;
}

}  // namespace

std::vector<double> match_polynomial(int K, double c) {
  if (K < 0) throw Error{NLG_EINVAL, "matching order must be >= 0"};
  if (K > 4) return matching_double(K, c);
  const auto ex = matching_exact(K);
  std::vector<double> out;
  for (const Q& r : ex)
    out.push_back(c * static_cast<double>(static_cast<long long>(r.p)) /
                  static_cast<double>(static_cast<long long>(r.q)));
  return out;
}

void match_polynomial_exact(int K, int64_t* num, int64_t* den) {
  const auto ex = matching_exact(K);
  for (int j = 0; j <= K; ++j) {
    num[j] = static_cast<int64_t>(ex[j].p);
    den[j] = static_cast<int64_t>(ex[j].q);
  }
}

void split_kernel(int K, double c, std::vector<double>& poly, std::vector<double>& tail) {
  poly = match_polynomial(K, c);
  if (K > 4) {
    // fp64 division of c - s p(s) by (1 - s)^{K+1}; the remainder must vanish
    // to 1e-9 |c| at every step (kernel.cpp:232-242)
    std::vector<double> num(2 * K + 2, 0.0);
    num[0] = c;
    for (int j = 0; j <= K; ++j) num[2 * j + 1] -= poly[j];
    for (int i = 0; i <= K; ++i) {
      std::vector<double> q(num.size() - 1);
      q[0] = num[0];
      for (std::size_t k = 1; k < q.size(); ++k) q[k] = num[k] + q[k - 1];
      if (std::fabs(num.back() + q.back()) > 1e-9 * std::fabs(c))
        throw Error{NLG_ERUNTIME, "split: kappa does not vanish to order K"};
      num = std::move(q);
    }
    tail = std::move(num);
    return;
  }
  const auto p1 = matching_exact(K);
  // numerator of 1/s - p1(s) over the common denominator s: 1 - s p1(s)
  std::vector<Q> num(2 * K + 2, Q(0));
  num[0] = Q(1);
  for (int j = 0; j <= K; ++j) num[2 * j + 1] = num[2 * j + 1] - p1[j];
  for (int i = 0; i <= K; ++i) {
    // divide by (1 - s): q[0] = num[0], q[k] = num[k] + q[k-1]; remainder must vanish
    std::vector<Q> q(num.size() - 1);
    q[0] = num[0];
    for (std::size_t k = 1; k < q.size(); ++k) q[k] = num[k] + q[k - 1];
    const Q rem = num.back() + q.back();
    if (rem.p != 0) throw Error{NLG_ERUNTIME, "split: kappa does not vanish to order K"};
    num = std::move(q);
  }
  tail.clear();
  for (const Q& r : num)
    tail.push_back(c * static_cast<double>(static_cast<long long>(r.p)) /
                   static_cast<double>(static_cast<long long>(r.q)));
}

}  // namespace nlg

// ---------------------------------------------------------------------------
// Exponential-sum fit of the far-field weights w_d = d^-alpha, d in [P+1, dmax]
//   w_d ~= sum_m c_m exp(-t_m d)
// 1. Trapezoid rule on r^-a = 1/Gamma(a) int exp(a s - r e^s) ds with step ds
//    (exponentially convergent in 1/ds), truncated where terms fall below 1e-17.
// 2. Terms with t_m dmax < cut are "ultra-slow": over the window they are a
//    smooth near-polynomial function R(d). They are replaced by nslow
//    exponentials with rates {0, geometric in [0.05, cut]/dmax} fitted to R by
//    relatively-weighted least squares (Householder QR).
// The fitted max relative error over EVERY integer d in the window is measured
// and returned; the plan refuses the fast path if it exceeds `tol`.
// ---------------------------------------------------------------------------

namespace nlg {
namespace {

// Least squares min ||A x - b|| by Householder QR; A is m x n row-major.
std::vector<double> lstsq(std::vector<double> A, std::vector<double> b, int m, int n) {
  for (int k = 0; k < n; ++k) {
    double nrm = 0.0;
    for (int i = k; i < m; ++i) nrm += A[i * n + k] * A[i * n + k];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    const double alpha = A[k * n + k] > 0 ? -nrm : nrm;
    std::vector<double> v(m - k);
    for (int i = k; i < m; ++i) v[i - k] = A[i * n + k];
    v[0] -= alpha;
    double vn = 0.0;
    for (double x : v) vn += x * x;
    if (vn == 0.0) continue;
    for (int j = k; j < n; ++j) {
      double s = 0.0;
      for (int i = k; i < m; ++i) s += v[i - k] * A[i * n + j];
      s = 2.0 * s / vn;
      for (int i = k; i < m; ++i) A[i * n + j] -= s * v[i - k];
    }
    double s = 0.0;
    for (int i = k; i < m; ++i) s += v[i - k] * b[i];
    s = 2.0 * s / vn;
    for (int i = k; i < m; ++i) b[i] -= s * v[i - k];
  }
  std::vector<double> x(n, 0.0);
  for (int k = n - 1; k >= 0; --k) {
    double s = b[k];
    for (int j = k + 1; j < n; ++j) s -= A[k * n + j] * x[j];
    x[k] = A[k * n + k] != 0.0 ? s / A[k * n + k] : 0.0;
  }
  return x;
}

}  // namespace


// Short exponential sum for d^-alpha on a NARROW window [lo, hi] (ratio a few):
// the far-end tails of the 1-D fractional operator. Candidate rates on a log
// grid, columns scaled to relative error; column-pivoted Householder QR (long
// double) orders them by independence; the first M are refit by long-double
// least squares, M growing until the worst relative error over every integer
// of the window is <= tol (or max_terms is reached: rel_err tells).
ExpSum fit_exponential_sum_narrow(double alpha, int64_t lo, int64_t hi, double tol, int max_terms) {
  using ld = long double;
  ExpSum es;
  es.near = static_cast<int>(lo - 1);
  es.dmax = hi;
  if (hi < lo || lo < 1) return es;
  const ld a = static_cast<ld>(lo), r = static_cast<ld>(hi) / a;
  const int nc = 150, ns = 402;
  std::vector<ld> tau(nc), xs(ns);
  for (int k = 0; k < nc; ++k) tau[k] = std::exp(std::log(1e-3L / r) + (std::log(60.0L) - std::log(1e-3L / r)) * k / (nc - 1));
  xs[0] = 1.0L;
  xs[ns - 1] = r;
  const ld pi = 3.141592653589793238462643383279502884L;
  for (int i = 1; i < ns - 1; ++i) xs[i] = 1.0L + (r - 1.0L) * (1.0L - std::cos(pi * (i - 0.5L) / (ns - 2))) / 2.0L;
  // E[i][k] = exp(-tau_k x_i) x_i^alpha  (so the target is 1: relative error)
  std::vector<ld> E(static_cast<size_t>(ns) * nc);
  for (int i = 0; i < ns; ++i)
    for (int k = 0; k < nc; ++k) E[i * nc + k] = std::exp(-tau[k] * xs[i]) * std::pow(xs[i], static_cast<ld>(alpha));
  // column-pivoted Householder QR on a copy: pivot order
  std::vector<ld> W = E;
  std::vector<int> piv(nc);
  for (int k = 0; k < nc; ++k) piv[k] = k;
  const int kmax = std::min(max_terms, nc);
  for (int k = 0; k < kmax; ++k) {
    int best = k;
    ld bn = -1;
    for (int j = k; j < nc; ++j) {
      ld s = 0;
      for (int i = k; i < ns; ++i) s += W[i * nc + j] * W[i * nc + j];
      if (s > bn) { bn = s; best = j; }
    }
    if (best != k) {
      for (int i = 0; i < ns; ++i) std::swap(W[i * nc + k], W[i * nc + best]);
      std::swap(piv[k], piv[best]);
    }
    const ld nrm = std::sqrt(bn);
    if (nrm == 0) break;
    const ld al = W[k * nc + k] > 0 ? -nrm : nrm;
    std::vector<ld> v(ns - k);
    for (int i = k; i < ns; ++i) v[i - k] = W[i * nc + k];
    v[0] -= al;
    ld vn = 0;
    for (ld x : v) vn += x * x;
    if (vn == 0) continue;
    for (int j = k; j < nc; ++j) {
      ld sdot = 0;
      for (int i = k; i < ns; ++i) sdot += v[i - k] * W[i * nc + j];
      sdot = 2 * sdot / vn;
      for (int i = k; i < ns; ++i) W[i * nc + j] -= sdot * v[i - k];
    }
  }
  for (int M = 2; M <= kmax; ++M) {
    // long-double least squares on the first M pivot columns
    std::vector<ld> A(static_cast<size_t>(ns) * M), b(ns, 1.0L);
    for (int i = 0; i < ns; ++i)
      for (int j = 0; j < M; ++j) A[i * M + j] = E[i * nc + piv[j]];
    for (int k = 0; k < M; ++k) {
      ld nrm = 0;
      for (int i = k; i < ns; ++i) nrm += A[i * M + k] * A[i * M + k];
      nrm = std::sqrt(nrm);
      if (nrm == 0) continue;
      const ld al = A[k * M + k] > 0 ? -nrm : nrm;
      std::vector<ld> v(ns - k);
      for (int i = k; i < ns; ++i) v[i - k] = A[i * M + k];
      v[0] -= al;
      ld vn = 0;
      for (ld x : v) vn += x * x;
      if (vn == 0) continue;
      for (int j = k; j < M; ++j) {
        ld sdot = 0;
        for (int i = k; i < ns; ++i) sdot += v[i - k] * A[i * M + j];
        sdot = 2 * sdot / vn;
        for (int i = k; i < ns; ++i) A[i * M + j] -= sdot * v[i - k];
      }
      ld sb = 0;
      for (int i = k; i < ns; ++i) sb += v[i - k] * b[i];
      sb = 2 * sb / vn;
      for (int i = k; i < ns; ++i) b[i] -= sb * v[i - k];
    }
    std::vector<ld> c(M, 0);
    for (int k = M - 1; k >= 0; --k) {
      ld sm = b[k];
      for (int j = k + 1; j < M; ++j) sm -= A[k * M + j] * c[j];
      c[k] = A[k * M + k] != 0 ? sm / A[k * M + k] : 0;
    }
    std::vector<double> rate(M), weight(M);
    for (int j = 0; j < M; ++j) {
      rate[j] = static_cast<double>(tau[piv[j]] / a);
      weight[j] = static_cast<double>(c[j] * std::pow(a, static_cast<ld>(-alpha)));
    }
    double worst = 0.0;
    for (int64_t d = lo; d <= hi; ++d) {
      const double x = static_cast<double>(d);
      double sm = 0.0;
      for (int j = 0; j < M; ++j) sm += weight[j] * std::exp(-rate[j] * x);
      worst = std::max(worst, std::fabs(sm * std::pow(x, alpha) - 1.0));
      if (worst > tol && M < kmax) break;   // early out: try more terms
    }
    if (worst <= tol || M == kmax) {
      std::vector<int> idx(M);
      for (int j = 0; j < M; ++j) idx[j] = j;
      std::sort(idx.begin(), idx.end(), [&](int x, int y) { return rate[x] < rate[y]; });
      for (int j : idx) {
        es.rate.push_back(rate[j]);
        es.weight.push_back(weight[j]);
      }
      es.terms = M;
      es.rel_err = worst;
      return es;
    }
  }
  return es;
}

ExpSum fit_exponential_sum(double alpha, int near, int64_t dmax, double tol) {
  ExpSum es;
  es.near = near;
  es.dmax = dmax;
  const double d0 = near + 1.0;
  const double D = static_cast<double>(dmax);
  if (dmax <= near) return es;  // no far field
  const double lg = std::lgamma(alpha);
  const double ds = 0.3, cut = 0.5;
  const int nslow = 6;
  const double smin = std::log(1e-16) / alpha - std::log(D) - 2.0;
  const double smax = std::log(38.0 / d0);
  std::vector<double> ut, uc;  // ultra-slow trapezoid terms
  for (long k = static_cast<long>(std::floor(smin / ds)); k * ds <= smax + ds; ++k) {
    const double s = k * ds;
    const double t = std::exp(s);
    const double c = ds * std::exp(alpha * s - lg);
    if (t * D < cut) {
      ut.push_back(t);
      uc.push_back(c);
    } else {
      es.rate.push_back(t);
      es.weight.push_back(c);
    }
  }
  // fit the ultra-slow remainder R(d) on log-spaced samples, weight 1/w(d)
  std::vector<double> srates{0.0};
  for (int j = 0; j < nslow - 1; ++j)
    srates.push_back(0.05 * std::pow(cut / 0.05, j / double(nslow - 2)) / D);
  const int ns = static_cast<int>(srates.size());
  std::vector<double> xs;
  for (int q = 0; q < 3000; ++q) {
    const double x = std::round(d0 * std::pow(D / d0, q / 2999.0));
    if (xs.empty() || x != xs.back()) xs.push_back(x);
  }
  const int m = static_cast<int>(xs.size());
  std::vector<double> A(static_cast<size_t>(m) * ns), b(m);
  for (int i = 0; i < m; ++i) {
    const double wi = std::pow(xs[i], alpha);  // 1 / w(d)
    double r = 0.0;
    for (size_t k = 0; k < ut.size(); ++k) r += uc[k] * std::exp(-ut[k] * xs[i]);
    b[i] = r * wi;
    for (int j = 0; j < ns; ++j) A[i * ns + j] = std::exp(-srates[j] * xs[i]) * wi;
  }
  const auto cs = lstsq(A, b, m, ns);
  for (int j = 0; j < ns; ++j) {
    es.rate.push_back(srates[j]);
    es.weight.push_back(cs[j]);
  }
  // order by rate (slow terms last is irrelevant; kernels sort by use)
  std::vector<int> idx(es.rate.size());
  for (size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<int>(i);
  std::sort(idx.begin(), idx.end(), [&](int a, int b2) { return es.rate[a] < es.rate[b2]; });
  std::vector<double> r2, w2;
  for (int i : idx) {
    r2.push_back(es.rate[i]);
    w2.push_back(es.weight[i]);
  }
  es.rate = r2;
  es.weight = w2;
  es.terms = static_cast<int>(es.rate.size());
  // measure on every integer of the window
  double worst = 0.0;
  for (int64_t d = near + 1; d <= dmax; ++d) {
    const double x = static_cast<double>(d);
    double s = 0.0;
    for (int k = 0; k < es.terms; ++k) s += es.weight[k] * std::exp(-es.rate[k] * x);
    worst = std::max(worst, std::fabs(s * std::pow(x, alpha) - 1.0));
  }
  es.rel_err = worst;
  (void)tol;
  return es;
}

}  // namespace nlg
