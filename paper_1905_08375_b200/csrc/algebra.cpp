// paper_1905_08375_b200/csrc/algebra.cpp — host-side kernel algebra (plan setup).
//
// match_polynomial: the even polynomial p(s) = sum_j c_j s^{2j} with
//   p^(m)(1) = gamma^(m)(1), m = 0..K, for gamma = c/s (kernel.cpp:26-51, 184-207):
//   sum_j ff(2j, m) c_j = c (-1)^m m!. Solved in exact rationals (K <= 6) so the
//   coefficients are the correctly rounded quotients the reference produces.
// split_kernel: kappa(s) = c/s - p(s) written as c (1-s)^{K+1} tail(s) / s
//   (kernel.cpp:209-245): tail = (1 - s p1(s)) / (1-s)^{K+1}, exact division.
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

}  // namespace

std::vector<double> match_polynomial(int K, double c) {
  if (K < 0) throw Error{NLG_EINVAL, "matching order must be >= 0"};
  if (K > 6) throw Error{NLG_EUNSUPPORTED, "matching order > 6 is not supported"};
  const auto ex = matching_exact(K);
  std::vector<double> out;
  for (const Q& r : ex)
    out.push_back(c * static_cast<double>(static_cast<long long>(r.p)) /
                  static_cast<double>(static_cast<long long>(r.q)));
  return out;
}

void split_kernel(int K, double c, std::vector<double>& poly, std::vector<double>& tail) {
  poly = match_polynomial(K, c);
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
