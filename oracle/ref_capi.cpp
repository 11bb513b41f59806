// oracle/ref_capi.cpp — C entry points into the COMPILED REFERENCE.
//
// TEST INFRASTRUCTURE ONLY: built by oracle/Makefile against the unmodified
// reference sources under /root/reference/proj/src into oracle/_ref/. Only
// tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
// --impl reference) load it, as the checker / the reference CPU arm. Nothing in
// the product links it.
//
// Every function calls the reference's public API only:
//   TruncatedOperator (operators.hpp:28-54), apply_truncated_dense (:58-62),
//   apply_smooth_dense (:66-70), apply_full_dense (:73-75), apply_split (:94-96),
//   match_polynomial / split (kernel.hpp:63-66), random_vector (bench.hpp:24),
//   assemble_dense_matrix (operators.hpp:79-81), solve_dirichlet / choose_method /
//   dense_direct_solve (solve.hpp:27-39).
// BASELINE-only features (fractional |r|^-alpha kernels, per-node delta(x),
// C(x) and (kappa(x)+kappa(y))/2 weighting) are expressed through the
// reference's own coefficient_fn hook (kernel.hpp:101) with an InverseS
// profile and a Constant horizon delta_max (SURVEY.md §8(c) "Feature envelope").
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "nonloc/bench.hpp"
#include "nonloc/kernel.hpp"
#include "nonloc/operators.hpp"
#include "nonloc/solve.hpp"
#include "nonloc/tree.hpp"

using namespace nonloc;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::domain_error*>(&e)) return 2;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 3;
  return 4;
}

KernelSpec make_spec(int dim, int family, int order, int horizon_kind,
                     double delta0, double coeff, int symmetry) {
  KernelSpec spec;
  spec.dim = dim;
  switch (family) {
    case 0: spec.profile = RadialProfile::inverse_s(); break;
    case 1: spec.profile = RadialProfile::conical(); break;
    case 2: spec.profile = RadialProfile::regularized(order); break;
    case 3: spec.profile = RadialProfile::truncated_polynomial(order); break;
    default: throw std::invalid_argument("unknown family");
  }
  spec.horizon = {horizon_kind == 0 ? HorizonKind::Constant : HorizonKind::GaussianBump, delta0};
  spec.coefficient_value = coeff;
  spec.symmetry = symmetry == 0 ? SymmetryClass::NonDivergence : SymmetryClass::Divergence;
  return spec;
}

double secs(std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_random_vector(int64_t n, uint64_t seed, double* out) {
  try {
    const auto v = random_vector(n, seed);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_match_polynomial(int K, double c, double* coeffs) {
  try {
    const auto p = match_polynomial(RadialProfile::inverse_s(c), K);
    for (int j = 0; j <= K; ++j) coeffs[j] = p.coeffs[j];
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_split(int K, double c, double* poly, double* tail, int* ntail) {
  try {
    const auto sk = split(RadialProfile::inverse_s(c), K);
    for (int j = 0; j <= K; ++j) poly[j] = sk.polynomial.coeffs[j];
    *ntail = static_cast<int>(sk.tail.size());
    for (std::size_t j = 0; j < sk.tail.size(); ++j) tail[j] = sk.tail[j];
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_kappa(int K, double c, int64_t n, const double* s, double* out) {
  try {
    const auto sk = split(RadialProfile::inverse_s(c), K);
    for (int64_t i = 0; i < n; ++i) out[i] = sk.kappa(s[i]);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// Fast truncated apply (Steps 1-3). counters = {recur_calls, step2_ops, step3_ops};
// times = {step1_seconds, apply_seconds (mean over reps)}.
int ref_truncated_fast(int dim, int n, int K, int horizon_kind, double delta0,
                       double coeff, const double* u, double* out,
                       int64_t* counters, double* times, int reps) {
  try {
    const Grid g = Grid::make(dim, n);
    const KernelSpec spec = make_spec(dim, 3, K, horizon_kind, delta0, coeff, 0);
    const auto t0 = std::chrono::steady_clock::now();
    TruncatedOperator op(spec, g);
    const auto t1 = std::chrono::steady_clock::now();
    std::vector<double> r;
    if (reps < 1) reps = 1;
    for (int k = 0; k < reps; ++k) r = op.apply(std::span<const double>(u, g.total));
    const auto t2 = std::chrono::steady_clock::now();
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    if (counters) {
      counters[0] = op.recur_calls();
      counters[1] = op.step2_ops() / reps;
      counters[2] = op.step3_ops() / reps;
    }
    if (times) { times[0] = secs(t0, t1); times[1] = secs(t1, t2) / reps; }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_truncated_dense(int dim, int n, int K, int horizon_kind, double delta0,
                        double coeff, int rule, int form, const double* u,
                        double* out, int64_t* pairs) {
  try {
    const Grid g = Grid::make(dim, n);
    const KernelSpec spec = make_spec(dim, 3, K, horizon_kind, delta0, coeff, 0);
    const auto r = apply_truncated_dense(
        spec, g, rule == 0 ? InclusionRule::Leaf : InclusionRule::Point,
        std::span<const double>(u, g.total),
        form == 0 ? ApplyForm::Mass : ApplyForm::Difference, pairs);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_smooth_dense(int dim, int n, int K, int horizon_kind, double delta0,
                     double coeff, const double* u, double* out, int64_t* pairs) {
  try {
    const Grid g = Grid::make(dim, n);
    const KernelSpec spec = make_spec(dim, 0, 0, horizon_kind, delta0, coeff, 0);
    const SplitKernel sk = split(spec.profile, K);
    const auto r = apply_smooth_dense(sk, spec, g, std::span<const double>(u, g.total), pairs);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// family: 0 InverseS, 1 Conical, 2 Regularized(order), 3 Truncated(order).
int ref_full_dense(int dim, int n, int family, int order, int horizon_kind,
                   double delta0, double coeff, int symmetry, const double* u,
                   double* out, int64_t* pairs) {
  try {
    const Grid g = Grid::make(dim, n);
    const KernelSpec spec = make_spec(dim, family, order, horizon_kind, delta0, coeff, symmetry);
    const auto r = apply_full_dense(spec, g, std::span<const double>(u, g.total), pairs);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// truncated: 0 FastLeafMass, 1 DensePointDifference (backend always Dense).
int ref_apply_split(int dim, int n, int K, int horizon_kind, double delta0,
                    double coeff, int truncated, const double* u, double* out) {
  try {
    const Grid g = Grid::make(dim, n);
    const KernelSpec spec = make_spec(dim, 0, 0, horizon_kind, delta0, coeff, 0);
    SplitApplyOptions opt;
    opt.backend = SmoothBackend::Dense;
    opt.truncated = truncated == 0 ? TruncatedPath::FastLeafMass : TruncatedPath::DensePointDifference;
    const auto r = apply_split(spec, g, K, std::span<const double>(u, g.total), opt);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// BASELINE operator through the reference's apply_full_dense (Point rule,
// Difference form, clipped exterior):
//   out_i = h^d sum_{k!=i, |y-x|<delta_i} C_i * kw(x,y) * |y-x|^-alpha (u_k-u_i)
// with kw = (kappa_i+kappa_k)/2 when kappa != NULL else 1. delta/cx are per-node
// arrays (row-major). Expressed as InverseS (c=1), Constant horizon delta_max,
// coefficient_fn(x,y) = [r<delta(x)] * omega(x,y) * delta_max^{d+1} * r, which
// eval_omega (kernel.cpp:275-287) turns back into omega(x,y).
int ref_full_dense_general(int dim, int n, const double* delta, double delta_max,
                           const double* cx, const double* kappa, double alpha,
                           const double* u, double* out, int64_t* pairs) {
  try {
    const Grid g = Grid::make(dim, n);
    KernelSpec spec;
    spec.dim = dim;
    spec.profile = RadialProfile::inverse_s(1.0);
    spec.horizon = {HorizonKind::Constant, delta_max};
    double dpow = delta_max;  // delta_max^{d+1}
    for (int j = 0; j < dim; ++j) dpow *= delta_max;
    const auto index_of = [g](const Point& p) {
      std::int64_t flat = 0;
      for (int j = 0; j < g.dim; ++j)
        flat = flat * g.n + static_cast<std::int64_t>(std::floor(p[j] * g.n));
      return flat;
    };
    spec.coefficient_fn = [=](const Point& x, const Point& y) {
      double r2 = 0.0;
      for (int j = 0; j < dim; ++j) { const double d = y[j] - x[j]; r2 += d * d; }
      const double r = std::sqrt(r2);
      const std::int64_t ix = index_of(x), iy = index_of(y);
      if (!(r < delta[ix])) return 0.0;
      double c = cx ? cx[ix] : 1.0;
      if (kappa) c *= 0.5 * (kappa[ix] + kappa[iy]);
      return c * std::pow(r, -alpha) * dpow * r;
    };
    const auto r = apply_full_dense(spec, g, std::span<const double>(u, g.total), pairs);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// Same operator as ref_full_dense_general, evaluated only at `targets` and
// split across `nthreads` std::threads: the per-target loop of
// apply_full_dense (operators.cpp:244-256, window_around :31-42 restated since
// it is file-local) around the reference's own eval_omega (kernel.cpp:275-287)
// with the same coefficient_fn. Used for the bounded CPU baseline at BASELINE
// sizes, where the whole-grid reference call would take hours.
int ref_full_dense_general_at(int dim, int n, const double* delta, double delta_max,
                              const double* cx, const double* kappa, double alpha,
                              const double* u, const int64_t* targets, int64_t ntargets,
                              double* out, int nthreads, int64_t* pairs_out) {
  try {
    const Grid g = Grid::make(dim, n);
    KernelSpec spec;
    spec.dim = dim;
    spec.profile = RadialProfile::inverse_s(1.0);
    spec.horizon = {HorizonKind::Constant, delta_max};
    double dpow = delta_max;
    for (int j = 0; j < dim; ++j) dpow *= delta_max;
    const auto index_of = [g](const Point& p) {
      std::int64_t flat = 0;
      for (int j = 0; j < g.dim; ++j)
        flat = flat * g.n + static_cast<std::int64_t>(std::floor(p[j] * g.n));
      return flat;
    };
    spec.coefficient_fn = [=](const Point& x, const Point& y) {
      double r2 = 0.0;
      for (int j = 0; j < dim; ++j) { const double d = y[j] - x[j]; r2 += d * d; }
      const double r = std::sqrt(r2);
      const std::int64_t ix = index_of(x), iy = index_of(y);
      if (!(r < delta[ix])) return 0.0;
      double c = cx ? cx[ix] : 1.0;
      if (kappa) c *= 0.5 * (kappa[ix] + kappa[iy]);
      return c * std::pow(r, -alpha) * dpow * r;
    };
    double hd = g.h;
    for (int j = 1; j < dim; ++j) hd *= g.h;
    if (nthreads < 1) nthreads = 1;
    std::vector<std::int64_t> pc(nthreads, 0);
    auto work = [&](int tid) {
      for (std::int64_t t = tid; t < ntargets; t += nthreads) {
        const std::int64_t i = targets[t];
        const Point x = node_position(g, i);
        std::int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        for (int j = 0; j < dim; ++j) {
          const double l = (x[j] - delta_max) / g.h - 1.0;
          const double h2 = (x[j] + delta_max) / g.h + 1.0;
          lo[j] = std::max<std::int64_t>(0, static_cast<std::int64_t>(std::floor(l)));
          hi[j] = std::min<std::int64_t>(g.n - 1, static_cast<std::int64_t>(std::ceil(h2)));
        }
        double acc = 0.0;
        std::int64_t k[3];
        for (k[0] = lo[0]; k[0] <= hi[0]; ++k[0])
          for (k[1] = lo[1]; k[1] <= hi[1]; ++k[1])
            for (k[2] = lo[2]; k[2] <= hi[2]; ++k[2]) {
              std::int64_t flat = 0;
              for (int j = 0; j < dim; ++j) flat = flat * g.n + k[j];
              if (flat == i) continue;
              Point y{};
              for (int j = 0; j < dim; ++j) y[j] = (static_cast<double>(k[j]) + 0.5) * g.h;
              const double w = eval_omega(spec, x, y);
              if (w == 0.0) continue;
              ++pc[tid];
              acc += w * (u[flat] - u[i]);
            }
        out[t] = hd * acc;
      }
    };
    std::vector<std::thread> th;
    for (int k = 1; k < nthreads; ++k) th.emplace_back(work, k);
    work(0);
    for (auto& x : th) x.join();
    if (pairs_out) {
      std::int64_t s = 0;
      for (auto v : pc) s += v;
      *pairs_out = s;
    }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}


// Dense matrix (row-major N x N) of the truncated operator (K, horizon, rule, form)
// or, for family >= 0 (full-operator profile), of apply_full_dense's operator.
int ref_assemble_dense(int dim, int n, int family, int order, int horizon_kind, double delta0,
                       double coeff, int symmetry, int rule, int form, double* a) {
  try {
    const Grid g = Grid::make(dim, n);
    const KernelSpec spec = make_spec(dim, family, order, horizon_kind, delta0, coeff, symmetry);
    const auto m = assemble_dense_matrix(spec, g, rule == 0 ? InclusionRule::Leaf : InclusionRule::Point,
                                         form == 0 ? ApplyForm::Mass : ApplyForm::Difference);
    std::memcpy(a, m.data(), sizeof(double) * m.size());
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// The reference's solve path of tools/nonloc_main.cpp:cmd_solve (lines 189-222):
// A = -L^P of the truncated K operator; choose_method(spec); CG through the
// fast TruncatedOperator (use_dense = 0) or the dense Leaf apply (use_dense = 1);
// CGNR through the assembled dense matrix and its transpose.
int ref_solve_truncated(int dim, int n, int K, int horizon_kind, double delta0, double coeff,
                        const double* f, double tol, int64_t max_iter, int use_dense, double* u,
                        int64_t* iterations, double* final_residual, int* converged, int* method) {
  try {
    const Grid g = Grid::make(dim, n);
    const KernelSpec spec = make_spec(dim, 3, K, horizon_kind, delta0, coeff, 0);
    const std::span<const double> fs(f, g.total);
    const SolveMethod m = choose_method(spec);
    SolveReport rep;
    if (m == SolveMethod::CG) {
      if (use_dense) {
        const auto apply = [&](std::span<const double> x) {
          auto out = apply_truncated_dense(spec, g, InclusionRule::Leaf, x);
          for (double& v : out) v = -v;
          return out;
        };
        rep = solve_dirichlet(apply, fs, tol, max_iter, SolveMethod::CG);
      } else {
        TruncatedOperator op(spec, g);
        const auto apply = [&](std::span<const double> x) {
          auto out = op.apply(x);
          for (double& v : out) v = -v;
          return out;
        };
        rep = solve_dirichlet(apply, fs, tol, max_iter, SolveMethod::CG);
      }
    } else {
      auto a = assemble_dense_matrix(spec, g, InclusionRule::Leaf, ApplyForm::Mass);
      for (double& v : a) v = -v;
      const int64_t N = g.total;
      const auto apply = [&](std::span<const double> x) {
        std::vector<double> out(N, 0.0);
        for (int64_t i = 0; i < N; ++i) {
          double acc = 0.0;
          for (int64_t j = 0; j < N; ++j) acc += a[i * N + j] * x[j];
          out[i] = acc;
        }
        return out;
      };
      const auto apply_t = [&](std::span<const double> x) {
        std::vector<double> out(N, 0.0);
        for (int64_t i = 0; i < N; ++i)
          for (int64_t j = 0; j < N; ++j) out[j] += a[i * N + j] * x[i];
        return out;
      };
      rep = solve_dirichlet(apply, fs, tol, max_iter, SolveMethod::CGNR, apply_t);
    }
    std::memcpy(u, rep.solution.data(), sizeof(double) * g.total);
    *iterations = rep.iterations;
    *final_residual = rep.final_residual;
    *converged = rep.converged ? 1 : 0;
    *method = m == SolveMethod::CG ? 0 : 1;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// dense_direct_solve (partial-pivot LU)
int ref_dense_direct_solve(int64_t n, const double* a, const double* rhs, double* x) {
  try {
    const auto r = dense_direct_solve(std::span<const double>(a, n * n), std::span<const double>(rhs, n));
    std::memcpy(x, r.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// Step-1 tree instruments (tree.hpp:31-53): panels of decompose_region for one
// ball (levels / indices, up to cap) and the recursion-call count.
int ref_decompose(int dim, int n, const double* center, double radius, int64_t cap, int* levels,
                  int64_t* indices, int64_t* npanels, int64_t* recur_calls) {
  try {
    const Tree t = build_tree(Grid::make(dim, n));
    const Point c{center[0], dim > 1 ? center[1] : 0.0, dim > 2 ? center[2] : 0.0};
    const Decomposition d = decompose_region(t, c, radius);
    *npanels = static_cast<int64_t>(d.panels.size());
    *recur_calls = d.recur_calls;
    for (int64_t k = 0; k < *npanels && k < cap; ++k) {
      levels[k] = d.panels[k].level;
      indices[k] = d.panels[k].index;
    }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_count_recur_calls(int dim, int n, const double* radii, int64_t* total) {
  try {
    const Grid g = Grid::make(dim, n);
    *total = count_recur_calls(build_tree(g), std::span<const double>(radii, g.total));
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// accumulate_moments (tree.hpp:46-48): all levels flattened level-major.
int ref_moments(int dim, int n, int K, const double* u, double* out, int64_t* adds) {
  try {
    const Grid g = Grid::make(dim, n);
    const Tree t = build_tree(g);
    const MomentTable m = accumulate_moments(t, std::span<const double>(u, g.total), K, adds);
    int64_t o = 0;
    for (const auto& lv : m.levels)
      for (double v : lv) out[o++] = v;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}
}  // extern "C"
