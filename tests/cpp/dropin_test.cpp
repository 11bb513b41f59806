// tests/cpp/dropin_test.cpp — the reference's own pinned cases, written against
// the drop-in C++ API (include/nonloc/*.hpp -> libnonloc_b200.so -> B200).
// Each case cites the reference test it mirrors. Exit status = failures.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "nonloc/bench.hpp"
#include "nonloc/operators.hpp"
#include "nonloc/solve.hpp"

using namespace nonloc;

static int failures = 0;
#define EXPECT(cond)                                                        \
  do {                                                                      \
    if (!(cond)) {                                                          \
      ++failures;                                                           \
      std::fprintf(stderr, "%s:%d: FAILED: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                       \
  } while (0)

static double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num = std::max(num, std::abs(a[i] - b[i]));
    den = std::max(den, std::abs(b[i]));
  }
  return den > 0 ? num / den : num;
}

static KernelSpec truncated(int dim, int K, HorizonKind kind, double d0) {
  KernelSpec s;
  s.dim = dim;
  s.profile = RadialProfile::truncated_polynomial(K);
  s.horizon = {kind, d0};
  return s;
}

int main() {
  // test_operators.cpp:55-87 — fast == dense Leaf rule
  {
    const Grid g = Grid::make(2, 64);
    const auto spec = truncated(2, 0, HorizonKind::Constant, 0.5);
    TruncatedOperator op(spec, g);
    const auto u = random_vector(g.total, 42);
    EXPECT(rel(op.apply(u), apply_truncated_dense(spec, g, InclusionRule::Leaf, u)) <= 1e-12);
  }
  {
    const Grid g = Grid::make(1, 2048);
    const auto spec = truncated(1, 3, HorizonKind::GaussianBump, 0.25);
    TruncatedOperator op(spec, g);
    const auto u = random_vector(g.total, 43);
    EXPECT(rel(op.apply(u), apply_truncated_dense(spec, g, InclusionRule::Leaf, u)) <= 1e-10);
  }
  {
    const Grid g = Grid::make(3, 8);
    const auto spec = truncated(3, 0, HorizonKind::Constant, 0.5);
    TruncatedOperator op(spec, g);
    const auto u = random_vector(g.total, 44);
    EXPECT(rel(op.apply(u), apply_truncated_dense(spec, g, InclusionRule::Leaf, u)) <= 1e-12);
  }
  // test_operators.cpp:48-53 — zero in, zero out
  {
    const Grid g = Grid::make(1, 64);
    TruncatedOperator op(truncated(1, 2, HorizonKind::Constant, 0.25), g);
    for (double v : op.apply(std::vector<double>(g.total, 0.0))) EXPECT(v == 0.0);
  }
  // test_operators.cpp:89-104 — linearity
  {
    const Grid g = Grid::make(1, 512);
    TruncatedOperator op(truncated(1, 2, HorizonKind::GaussianBump, 0.25), g);
    const auto u = random_vector(g.total, 1), v = random_vector(g.total, 2);
    std::vector<double> w(g.total);
    for (std::int64_t i = 0; i < g.total; ++i) w[i] = 0.7 * u[i] - 1.9 * v[i];
    const auto fu = op.apply(u), fv = op.apply(v), fw = op.apply(w);
    double sc = 0;
    for (double x : fw) sc = std::max(sc, std::abs(x));
    for (std::int64_t i = 0; i < g.total; ++i) EXPECT(std::abs(fw[i] - (0.7 * fu[i] - 1.9 * fv[i])) <= 1e-12 * sc);
  }
  // test_operators.cpp:136-177 — smooth + truncated(Point, Difference) == full
  {
    const Grid g = Grid::make(1, 256);
    KernelSpec spec;
    spec.profile = RadialProfile::inverse_s();
    spec.horizon = {HorizonKind::Constant, 0.25};
    const SplitKernel sk = split(spec.profile, 2);
    for (double v : apply_smooth_dense(sk, spec, g, std::vector<double>(g.total, 3.25))) EXPECT(v == 0.0);
    const auto u = random_vector(g.total, 17);
    const auto sm = apply_smooth_dense(sk, spec, g, u);
    const auto tr = apply_truncated_dense(truncated(1, 2, HorizonKind::Constant, 0.25), g, InclusionRule::Point, u,
                                          ApplyForm::Difference);
    std::vector<double> sum(g.total);
    for (std::int64_t i = 0; i < g.total; ++i) sum[i] = sm[i] + tr[i];
    EXPECT(rel(sum, apply_full_dense(spec, g, u)) <= 1e-12);
    SplitApplyOptions opt;
    opt.truncated = TruncatedPath::DensePointDifference;
    EXPECT(rel(apply_split(spec, g, 2, u, opt), apply_full_dense(spec, g, u)) <= 1e-12);
    opt.backend = SmoothBackend::Hodlr;
    bool threw = false;
    try {
      apply_split(spec, g, 2, u, opt);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    EXPECT(threw);
  }
  // test_operators.cpp:235-246 — full operator annihilates constants (bump)
  for (int dim = 1; dim <= 2; ++dim) {
    const Grid g = Grid::make(dim, dim == 1 ? 256 : 16);
    KernelSpec spec;
    spec.dim = dim;
    spec.profile = RadialProfile::inverse_s();
    spec.horizon = {HorizonKind::GaussianBump, 0.25};
    for (double v : apply_full_dense(spec, g, std::vector<double>(g.total, 1.0))) EXPECT(std::abs(v) <= 1e-12);
  }
  // test_operators.cpp:248-285 — local limit: M2 = 1 (+-2%), linear u -> 0
  {
    const Grid g = Grid::make(1, 1024);
    const auto probe = local_limit_probe(RadialProfile::inverse_s(), 0.125, g);
    double best = 1e9, val = 0;
    for (std::size_t i = 0; i < probe.interior.size(); ++i) {
      const double x = (probe.interior[i] + 0.5) * g.h;
      if (std::abs(x - 0.5) < best) {
        best = std::abs(x - 0.5);
        val = probe.values[i];
      }
    }
    EXPECT(std::abs(val - 1.0) <= 0.02 * 2.0);
  }
  // test_kernel.cpp:95-110 — matching coefficients, exact rationals
  {
    const auto p3 = match_polynomial(RadialProfile::inverse_s(), 3);
    EXPECT(p3.coeffs[0] == 35.0 / 16.0 && p3.coeffs[3] == -5.0 / 16.0);
    EXPECT(p3.exact.size() == 4 && p3.exact[0].num == 35 && p3.exact[0].den == 16);
    EXPECT(std::abs(second_moment(RadialProfile::inverse_s()) - 1.0) <= 1e-9);
  }
  // geometry.cpp:13-16 / test_geometry.cpp:64-66 — error behaviour
  {
    bool t1 = false, t2 = false;
    try { (void)Grid::make(1, 3); } catch (const std::invalid_argument&) { t1 = true; }
    try { (void)node_position(Grid::make(1, 4), 4); } catch (const std::out_of_range&) { t2 = true; }
    EXPECT(t1 && t2);
  }
  // bench.cpp:34-72 — the conformance harness
  {
    const auto rec = run_apply_case(truncated(2, 0, HorizonKind::Constant, 0.25), Grid::make(2, 128), 7);
    EXPECT(rec.max_rel_err_vs_dense <= 1e-10 && rec.dense_pairs > 0);
  }
  std::printf("[dropin] failures: %d\n", failures);

  // ---- test_solve.cpp:47-170 through the drop-in solve.hpp ----
  {
    const std::vector<double> f0(64, 0.0);
    const auto rep = solve_dirichlet([](std::span<const double> u) { return std::vector<double>(u.begin(), u.end()); },
                                     f0, 1e-10, 100);
    EXPECT(rep.converged && rep.iterations == 0);
  }
  {
    const Grid g = Grid::make(1, 128);
    const auto a = assemble_dense_matrix(truncated(1, 1, HorizonKind::Constant, 0.25), g, InclusionRule::Leaf,
                                         ApplyForm::Mass);
    double num = 0.0, den = 0.0;
    for (std::int64_t i = 0; i < g.total; ++i)
      for (std::int64_t j = 0; j < g.total; ++j) {
        const double d = a[i * g.total + j] - a[j * g.total + i];
        num += d * d;
        den += a[i * g.total + j] * a[i * g.total + j];
      }
    EXPECT(std::sqrt(num) <= 1e-12 * std::sqrt(den));   // test_solve.cpp:60-71
  }
  auto manufactured = [](const Grid& g) {
    std::vector<double> u(g.total);
    for (std::int64_t i = 0; i < g.total; ++i) {
      const double x = (i + 0.5) * g.h;
      u[i] = std::sin(2.0 * 3.14159265358979323846 * x) * x * (1.0 - x);
    }
    return u;
  };
  auto negate = [](std::vector<double> v) {
    for (double& x : v) x = -x;
    return v;
  };
  {
    const Grid g = Grid::make(1, 512);
    const KernelSpec spec = truncated(1, 0, HorizonKind::Constant, 0.25);
    const auto ustar = manufactured(g);
    const auto f = negate(apply_truncated_dense(spec, g, InclusionRule::Leaf, ustar));
    const auto apply = [&](std::span<const double> u) {
      return negate(apply_truncated_dense(spec, g, InclusionRule::Leaf, u));
    };
    const auto rep = solve_dirichlet(apply, f, 1e-10, 10 * g.total);   // dense matvec subcase
    EXPECT(rep.converged && rep.final_residual <= 1e-10);
    EXPECT(rel(rep.solution, ustar) <= 1e-8);
    TruncatedOperator op(spec, g);
    const auto rep2 = solve_dirichlet(op, f, 1e-10, 10 * g.total);    // device-resident, fast apply
    EXPECT(rep2.method == SolveMethod::CG && rep2.converged);
    EXPECT(rel(rep2.solution, ustar) <= 1e-8);
    auto a = assemble_dense_matrix(spec, g, InclusionRule::Leaf, ApplyForm::Mass);
    for (double& v : a) v = -v;
    EXPECT(rel(rep2.solution, dense_direct_solve(a, f)) <= 1e-8);
  }
  {
    const Grid g = Grid::make(1, 256);
    const KernelSpec spec = truncated(1, 0, HorizonKind::GaussianBump, 0.25);
    EXPECT(choose_method(spec) == SolveMethod::CGNR);
    const auto ustar = manufactured(g);
    const auto f = negate(apply_truncated_dense(spec, g, InclusionRule::Leaf, ustar));
    auto a = assemble_dense_matrix(spec, g, InclusionRule::Leaf, ApplyForm::Mass);
    for (double& v : a) v = -v;
    TruncatedOperator op(spec, g);
    const auto rep = solve_dirichlet(op, f, 1e-10, 10 * g.total);     // CGNR, GPU transpose
    EXPECT(rep.method == SolveMethod::CGNR && rep.converged);
    EXPECT(rel(rep.solution, dense_direct_solve(a, f)) <= 1e-6);
    bool threw = false;
    try {
      (void)solve_dirichlet([&](std::span<const double> u) { return std::vector<double>(u.begin(), u.end()); }, f,
                            1e-10, 10, SolveMethod::CGNR);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    EXPECT(threw);
  }
  {
    const Grid g = Grid::make(1, 128);
    TruncatedOperator op(truncated(1, 0, HorizonKind::Constant, 0.25), g);
    const auto f = negate(apply_truncated_dense(op.spec(), g, InclusionRule::Leaf, manufactured(g)));
    const auto rep = solve_dirichlet(op, f, 1e-14, 2);
    EXPECT(!rep.converged && rep.iterations == 2);                  // test_solve.cpp:147-158
    std::vector<double> fn(16, 1.0);
    bool threw = false;
    try {
      (void)solve_dirichlet([](std::span<const double> u) {
        std::vector<double> out(u.begin(), u.end());
        out[0] = std::nan("");
        return out;
      }, fn, 1e-10, 10);
    } catch (const std::runtime_error&) {
      threw = true;
    }
    EXPECT(threw);                                                  // test_solve.cpp:160-170
  }
  return failures;
}
