// paper_1905_08375_b200/csrc/nonloc_api.cpp — the reference's C++ operator API
// (include/nonloc/*.hpp) implemented over the C-ABI (include/nlgpu.h).
//
// Host-side pieces (geometry predicates, kernel algebra, horizon fields) are
// small restatements of the reference semantics cited per function; every
// apply goes to the GPU. Status codes map back to the reference's exceptions
// (SURVEY §8(b)): EINVAL/EUNSUPPORTED -> invalid_argument, EDOMAIN ->
// domain_error, ERANGE -> out_of_range, everything else -> runtime_error.
#include <chrono>
#include <cmath>
#include <functional>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "nlgpu.h"
#include "nonloc/bench.hpp"
#include "nonloc/geometry.hpp"
#include "nonloc/kernel.hpp"
#include "nonloc/operators.hpp"
#include "nonloc/solve.hpp"
#include "nonloc/tree.hpp"

namespace nonloc {

namespace {

void check(nlg_status st) {
  if (st == NLG_OK) return;
  const std::string msg = nlg_last_error();
  switch (st) {
    case NLG_EINVAL:
    case NLG_EUNSUPPORTED: throw std::invalid_argument(msg);
    case NLG_EDOMAIN: throw std::domain_error(msg);
    case NLG_ERANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

}  // namespace

// ---- geometry (geometry.cpp:9-97) -----------------------------------------

bool is_power_of_two(int n) { return n > 0 && (n & (n - 1)) == 0; }

Grid Grid::make(int dim, int n) {
  if (dim < 1 || dim > 3) throw std::invalid_argument("grid dimension must be 1, 2 or 3");
  if (n < 2 || !is_power_of_two(n))
    throw std::invalid_argument("grid n must be a power of two >= 2, got " + std::to_string(n));
  Grid g;
  g.dim = dim;
  g.n = n;
  g.h = 1.0 / n;
  g.total = 1;
  for (int j = 0; j < dim; ++j) g.total *= n;
  return g;
}

int Grid::levels() const {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

Aabb panel_bounds(int dim, const PanelId& id) {
  const std::int64_t per = std::int64_t{1} << id.level;
  const double w = 1.0 / static_cast<double>(per);
  Aabb b;
  std::int64_t rest = id.index;
  for (int j = dim - 1; j >= 0; --j) {
    const std::int64_t k = rest % per;
    rest /= per;
    b.min[j] = static_cast<double>(k) * w;
    b.max[j] = static_cast<double>(k + 1) * w;
  }
  return b;
}

bool cube_inside_ball(int dim, const Aabb& box, const Point& c, double r) {
  const double r2 = r * r;   // closed ball, every corner
  for (int corner = 0; corner < (1 << dim); ++corner) {
    double d2 = 0.0;
    for (int j = 0; j < dim; ++j) {
      const double d = ((corner >> j) & 1 ? box.max[j] : box.min[j]) - c[j];
      d2 += d * d;
    }
    if (d2 > r2) return false;
  }
  return true;
}

bool cube_intersects_ball(int dim, const Aabb& box, const Point& c, double r) {
  double dmin = 0.0;   // clamp distance, strict comparison (grazing is out)
  for (int j = 0; j < dim; ++j) {
    if (box.min[j] > c[j]) {
      const double d = box.min[j] - c[j];
      dmin += d * d;
    } else if (box.max[j] < c[j]) {
      const double d = box.max[j] - c[j];
      dmin += d * d;
    }
  }
  return dmin < r * r;
}

std::array<std::int64_t, 3> node_multi_index(const Grid& g, std::int64_t flat) {
  if (flat < 0 || flat >= g.total) throw std::out_of_range("node index out of range");
  std::array<std::int64_t, 3> k{};
  for (int j = g.dim - 1; j >= 0; --j) {
    k[j] = flat % g.n;
    flat /= g.n;
  }
  return k;
}

Point node_position(const Grid& g, std::int64_t flat) {
  const auto k = node_multi_index(g, flat);
  Point x{};
  for (int j = 0; j < g.dim; ++j) x[j] = (static_cast<double>(k[j]) + 0.5) * g.h;
  return x;
}

// ---- kernel algebra (kernel.cpp:106-287) ----------------------------------

double MatchedPolynomial::operator()(double s) const {
  const double t = s * s;
  double acc = 0.0;
  for (auto it = coeffs.rbegin(); it != coeffs.rend(); ++it) acc = acc * t + *it;
  return acc;
}

double SplitKernel::kappa(double s) const {
  s = std::abs(s);
  if (s == 0.0) throw std::domain_error("kappa is singular at s = 0");
  if (s >= 1.0) return 0.0;
  if (s < 0.5) return scale / s - polynomial(s);
  const double u = 1.0 - s;
  double f = 1.0;
  for (int i = 0; i <= polynomial.order; ++i) f *= u;
  double acc = 0.0;
  for (auto it = tail.rbegin(); it != tail.rend(); ++it) acc = acc * s + *it;
  return f * acc / s;
}

RadialProfile RadialProfile::inverse_s(double c) {
  RadialProfile p;
  p.family = ProfileFamily::InverseS;
  p.c = c;
  return p;
}

RadialProfile RadialProfile::conical(double c) {
  RadialProfile p = inverse_s(c);
  p.family = ProfileFamily::ConicalInverseS;
  return p;
}

RadialProfile RadialProfile::regularized(int k, double c) {
  RadialProfile p = inverse_s(c);
  p.family = ProfileFamily::Regularized;
  p.order = k;
  p.split_data = std::make_shared<SplitKernel>(split(inverse_s(c), k));
  return p;
}

RadialProfile RadialProfile::truncated_polynomial(int K, double c) {
  RadialProfile p = inverse_s(c);
  p.family = ProfileFamily::PolynomialTruncated;
  p.order = K;
  p.poly = std::make_shared<MatchedPolynomial>(match_polynomial(inverse_s(c), K));
  return p;
}

bool RadialProfile::singular_at_origin() const { return family != ProfileFamily::PolynomialTruncated; }

double eval_profile(const RadialProfile& p, double s) {
  s = std::abs(s);
  if (s >= 1.0) return 0.0;
  switch (p.family) {
    case ProfileFamily::InverseS:
      if (s == 0.0) throw std::domain_error("profile is singular at s = 0");
      return p.c / s;
    case ProfileFamily::ConicalInverseS:
      if (s == 0.0) throw std::domain_error("profile is singular at s = 0");
      return p.c / s * (1.0 - s);
    case ProfileFamily::Regularized: return p.split_data->kappa(s);
    case ProfileFamily::PolynomialTruncated: return (*p.poly)(s);
  }
  return 0.0;
}

MatchedPolynomial match_polynomial(const RadialProfile& profile, int K) {
  if (profile.family != ProfileFamily::InverseS)
    throw std::invalid_argument("match_polynomial requires the InverseS profile");
  if (K < 0) throw std::invalid_argument("matching order must be >= 0");
  MatchedPolynomial m;
  m.order = K;
  m.coeffs.resize(K + 1);
  check(nlg_match_polynomial(K, profile.c, m.coeffs.data()));
  if (profile.c == 1.0 && K <= 4) {
    std::vector<int64_t> num(K + 1), den(K + 1);
    check(nlg_match_polynomial_exact(K, num.data(), den.data()));
    for (int j = 0; j <= K; ++j) m.exact.push_back({num[j], den[j]});
  }
  return m;
}

SplitKernel split(const RadialProfile& profile, int K) {
  if (profile.family != ProfileFamily::InverseS)
    throw std::invalid_argument("match_polynomial requires the InverseS profile");
  if (K < 0) throw std::invalid_argument("matching order must be >= 0");
  SplitKernel sk;
  sk.scale = profile.c;
  sk.polynomial = match_polynomial(profile, K);
  std::vector<double> poly(K + 1), tail(K + 2);
  int nt = 0;
  check(nlg_split(K, profile.c, poly.data(), tail.data(), &nt));
  sk.tail.assign(tail.begin(), tail.begin() + nt);
  return sk;
}

namespace {
double simpson(const std::function<double(double)>& f, double a, double b, double fa, double fm, double fb,
               double whole, double eps, int depth) {
  const double m = 0.5 * (a + b), lm = 0.5 * (a + m), rm = 0.5 * (m + b);
  const double flm = f(lm), frm = f(rm);
  const double left = (m - a) / 6.0 * (fa + 4.0 * flm + fm);
  const double right = (b - m) / 6.0 * (fm + 4.0 * frm + fb);
  const double err = left + right - whole;
  if (depth <= 0 || std::abs(err) <= 15.0 * eps) return left + right + err / 15.0;
  return simpson(f, a, m, fa, flm, fm, left, 0.5 * eps, depth - 1) +
         simpson(f, m, b, fm, frm, fb, right, 0.5 * eps, depth - 1);
}
}  // namespace

double second_moment(const RadialProfile& profile) {
  // M2 = 2 int_0^1 s^2 gamma(s) ds (kernel.cpp:247-253), adaptive Simpson
  const std::function<double(double)> f = [&](double s) { return s <= 0.0 ? 0.0 : s * s * eval_profile(profile, s); };
  const double fa = f(0.0), fb = f(1.0), fm = f(0.5);
  const double whole = (fa + 4.0 * fm + fb) / 6.0;
  return 2.0 * simpson(f, 0.0, 1.0, fa, fm, fb, whole, 1e-11 * std::max(std::abs(whole), 1e-3), 40);
}

double HorizonField::operator()(const Point& x) const {
  if (kind == HorizonKind::Constant) return delta0;
  const double d = x[0] - 0.5;
  return delta0 * (1.0 + std::exp(-20.0 * d * d));
}

double HorizonField::max_radius() const { return kind == HorizonKind::Constant ? delta0 : 2.0 * delta0; }

double KernelSpec::coefficient(const Point& x, const Point& y) const {
  return coefficient_fn ? coefficient_fn(x, y) : coefficient_value;
}

double KernelSpec::horizon_at(const Point& x, const Point& y) const {
  return symmetry == SymmetryClass::Divergence ? 0.5 * (horizon(x) + horizon(y)) : horizon(x);
}

double eval_omega(const KernelSpec& spec, const Point& x, const Point& y) {
  double r2 = 0.0;
  for (int j = 0; j < spec.dim; ++j) {
    const double d = y[j] - x[j];
    r2 += d * d;
  }
  const double r = std::sqrt(r2);
  const double delta = spec.horizon_at(x, y);
  if (r >= delta) return 0.0;
  double dpow = delta * delta;
  for (int j = 0; j < spec.dim; ++j) dpow *= delta;
  return spec.coefficient(x, y) / dpow * eval_profile(spec.profile, r / delta);
}

// ---- operators over the C-ABI ---------------------------------------------

double ball_volume(int dim, double r) {
  switch (dim) {
    case 1: return 2.0 * r;
    case 2: return std::numbers::pi * r * r;
    case 3: return 4.0 / 3.0 * std::numbers::pi * r * r * r;
    default: throw std::invalid_argument("ball_volume: dim must be 1, 2 or 3");
  }
}

namespace {

// Host arrays a plan reads at creation (delta_ / coeff_ of operators.cpp:119-120).
struct NodeArrays {
  std::vector<double> delta, coeff, kappa, poly, tail;
};

nlg_desc make_desc(const KernelSpec& spec, const Grid& grid, NodeArrays& na) {
  if (spec.dim != grid.dim) throw std::invalid_argument("spec/grid dimension mismatch");
  nlg_desc d{};
  d.dim = grid.dim;
  d.n = grid.n;
  d.delta0 = spec.horizon.delta0;
  d.coeff0 = spec.coefficient_value;
  d.c = spec.profile.c;
  d.divergence = spec.symmetry == SymmetryClass::Divergence;
  if (spec.horizon.kind != HorizonKind::Constant || spec.coefficient_fn) {
    if (spec.horizon.kind != HorizonKind::Constant) na.delta.resize(grid.total);
    if (spec.coefficient_fn) na.coeff.resize(grid.total);
    for (std::int64_t i = 0; i < grid.total; ++i) {
      const Point x = node_position(grid, i);
      if (!na.delta.empty()) na.delta[i] = spec.horizon(x);
      if (!na.coeff.empty()) na.coeff[i] = spec.coefficient_at(x);
    }
  }
  if (!spec.kappa_nodes.empty()) {
    if (static_cast<std::int64_t>(spec.kappa_nodes.size()) != grid.total)
      throw std::invalid_argument("kappa_nodes size does not match grid");
    na.kappa = spec.kappa_nodes;
  }
  d.delta = na.delta.empty() ? nullptr : na.delta.data();
  d.coeff = na.coeff.empty() ? nullptr : na.coeff.data();
  d.kappa = na.kappa.empty() ? nullptr : na.kappa.data();
  return d;
}

void set_profile(nlg_desc& d, const RadialProfile& p, NodeArrays& na) {
  switch (p.family) {
    case ProfileFamily::InverseS: d.family = NLG_INVERSE_S; break;
    case ProfileFamily::ConicalInverseS: d.family = NLG_CONICAL; break;
    case ProfileFamily::Regularized:
      d.family = NLG_KAPPA;
      na.poly = p.split_data->polynomial.coeffs;
      na.tail = p.split_data->tail;
      d.order = p.split_data->polynomial.order;
      d.c = p.split_data->scale;
      break;
    case ProfileFamily::PolynomialTruncated:
      d.family = NLG_TRUNCATED;
      na.poly = p.poly->coeffs;
      break;
  }
  d.poly = na.poly.empty() ? nullptr : na.poly.data();
  d.npoly = static_cast<int>(na.poly.size());
  d.tail = na.tail.empty() ? nullptr : na.tail.data();
  d.ntail = static_cast<int>(na.tail.size());
}

struct PlanGuard {
  nlg_plan* p = nullptr;
  ~PlanGuard() { nlg_plan_destroy(p); }
};

std::vector<double> run_direct(const nlg_desc& d, std::span<const double> u, std::int64_t* pair_count,
                               std::int64_t total) {
  if (static_cast<std::int64_t>(u.size()) != total) throw std::invalid_argument("u size does not match grid");
  PlanGuard g;
  check(nlg_plan_create(&d, &g.p));
  std::vector<double> out(total);
  int64_t pairs = 0;
  check(nlg_apply_direct(g.p, u.data(), out.data(), &pairs));
  if (pair_count) *pair_count += pairs;
  return out;
}

void require_truncated(const KernelSpec& spec) {
  if (spec.profile.family != ProfileFamily::PolynomialTruncated)
    throw std::invalid_argument("operation requires a PolynomialTruncated profile");
}

}  // namespace

TruncatedOperator::TruncatedOperator(const KernelSpec& spec, const Grid& grid) : spec_(spec), grid_(grid) {
  require_truncated(spec);
  if (spec.symmetry != SymmetryClass::NonDivergence)
    throw std::invalid_argument("the fast path is defined for the non-divergence form");
  const int K = spec.profile.order;
  if (grid.dim >= 2 && K != 0) throw std::invalid_argument("K > 0 is supported in 1d only");
  if (grid.dim == 1 && K > 3) throw std::invalid_argument("K <= 3 in 1d");
  make_plan();
}

void TruncatedOperator::make_plan() {
  NodeArrays na;
  nlg_desc d = make_desc(spec_, grid_, na);
  set_profile(d, spec_.profile, na);
  d.route = NLG_ROUTE_TRUNCATED;
  d.rule = NLG_LEAF;
  d.form = NLG_MASS;
  check(nlg_plan_create(&d, &plan_));
}

TruncatedOperator::~TruncatedOperator() { nlg_plan_destroy(plan_); }

TruncatedOperator::TruncatedOperator(const TruncatedOperator& o)
    : spec_(o.spec_), grid_(o.grid_), applies_(o.applies_), tree_(o.tree_), have_totals_(o.have_totals_),
      recur_(o.recur_), panels_(o.panels_), decomp_(o.decomp_) {
  make_plan();
}

TruncatedOperator& TruncatedOperator::operator=(const TruncatedOperator& o) {
  if (this != &o) {
    TruncatedOperator tmp(o);
    *this = std::move(tmp);
  }
  return *this;
}

TruncatedOperator::TruncatedOperator(TruncatedOperator&& o) noexcept
    : spec_(std::move(o.spec_)), grid_(o.grid_), plan_(o.plan_), applies_(o.applies_), tree_(o.tree_),
      have_totals_(o.have_totals_), recur_(o.recur_), panels_(o.panels_), decomp_(std::move(o.decomp_)) {
  o.plan_ = nullptr;
}

TruncatedOperator& TruncatedOperator::operator=(TruncatedOperator&& o) noexcept {
  if (this != &o) {
    nlg_plan_destroy(plan_);
    spec_ = std::move(o.spec_);
    grid_ = o.grid_;
    plan_ = o.plan_;
    o.plan_ = nullptr;
    applies_ = o.applies_;
    tree_ = std::move(o.tree_);
    have_totals_ = o.have_totals_;
    recur_ = o.recur_;
    panels_ = o.panels_;
    decomp_ = std::move(o.decomp_);
  }
  return *this;
}

std::vector<double> TruncatedOperator::apply(std::span<const double> u) {
  if (static_cast<std::int64_t>(u.size()) != grid_.total) throw std::invalid_argument("u size does not match grid");
  std::vector<double> out(grid_.total);
  check(nlg_apply_fast(plan_, u.data(), out.data()));
  ++applies_;
  return out;
}

std::vector<double> apply_truncated_dense(const KernelSpec& spec, const Grid& grid, InclusionRule rule,
                                          std::span<const double> u, ApplyForm form, std::int64_t* pair_count) {
  require_truncated(spec);
  NodeArrays na;
  nlg_desc d = make_desc(spec, grid, na);
  set_profile(d, spec.profile, na);
  d.route = NLG_ROUTE_TRUNCATED;
  d.rule = rule == InclusionRule::Leaf ? NLG_LEAF : NLG_POINT;
  d.form = form == ApplyForm::Mass ? NLG_MASS : NLG_DIFFERENCE;
  d.divergence = 0;
  return run_direct(d, u, pair_count, grid.total);
}

std::vector<double> apply_smooth_dense(const SplitKernel& sk, const KernelSpec& spec, const Grid& grid,
                                       std::span<const double> u, std::int64_t* pair_count) {
  NodeArrays na;
  nlg_desc d = make_desc(spec, grid, na);
  na.poly = sk.polynomial.coeffs;
  na.tail = sk.tail;
  d.family = NLG_KAPPA;
  d.route = NLG_ROUTE_SMOOTH;
  d.poly = na.poly.data();
  d.npoly = static_cast<int>(na.poly.size());
  d.tail = na.tail.data();
  d.ntail = static_cast<int>(na.tail.size());
  d.order = sk.polynomial.order;
  d.c = sk.scale;
  d.rule = NLG_POINT;
  d.form = NLG_DIFFERENCE;
  d.divergence = 0;
  return run_direct(d, u, pair_count, grid.total);
}

std::vector<double> apply_full_dense(const KernelSpec& spec, const Grid& grid, std::span<const double> u,
                                     std::int64_t* pair_count) {
  NodeArrays na;
  nlg_desc d = make_desc(spec, grid, na);
  set_profile(d, spec.profile, na);
  d.route = NLG_ROUTE_FULL;
  d.rule = NLG_POINT;
  d.form = NLG_DIFFERENCE;
  d.reach = spec.horizon.max_radius();
  return run_direct(d, u, pair_count, grid.total);
}

// ---- Step-1 tree API (tree.hpp) over the host instruments in libnlgpu -------

std::int64_t Tree::panels_at(int level) const { return std::int64_t{1} << (grid.dim * level); }

PanelId Tree::child(const PanelId& id, int which) const {
  const std::int64_t per = std::int64_t{1} << id.level;
  std::int64_t k[3] = {0, 0, 0}, rest = id.index;
  for (int j = grid.dim - 1; j >= 0; --j) {
    k[j] = rest % per;
    rest /= per;
  }
  std::int64_t f = 0;
  for (int j = 0; j < grid.dim; ++j) f = f * (2 * per) + (2 * k[j] + ((which >> j) & 1));
  return {id.level + 1, f};
}

PanelId Tree::parent(const PanelId& id) const {
  if (id.level == 0) throw std::invalid_argument("root has no parent");
  const std::int64_t per = std::int64_t{1} << id.level;
  std::int64_t k[3] = {0, 0, 0}, rest = id.index;
  for (int j = grid.dim - 1; j >= 0; --j) {
    k[j] = rest % per;
    rest /= per;
  }
  std::int64_t f = 0;
  for (int j = 0; j < grid.dim; ++j) f = f * (per / 2) + k[j] / 2;
  return {id.level - 1, f};
}

Tree build_tree(const Grid& grid) {
  if (!is_power_of_two(grid.n)) throw std::invalid_argument("tree requires n to be a power of two");
  Tree t;
  t.grid = grid;
  t.depth = grid.levels();
  return t;
}

Decomposition decompose_region(const Tree& tree, const Point& center, double radius) {
  Decomposition d;
  d.center = center;
  d.radius = radius;
  std::int64_t cap = 4096;
  for (;;) {
    std::vector<int> lv(cap);
    std::vector<int64_t> ix(cap);
    int64_t np = 0, rc = 0;
    check(nlg_tree_decompose(tree.grid.dim, tree.grid.n, center.data(), radius, cap, lv.data(), ix.data(), &np,
                             &rc));
    if (np > cap) {
      cap = np;
      continue;
    }
    d.recur_calls = rc;
    d.panels.resize(np);
    for (int64_t k = 0; k < np; ++k) d.panels[k] = {lv[k], ix[k]};
    return d;
  }
}

MomentTable accumulate_moments(const Tree& tree, std::span<const double> u, int K, std::int64_t* add_count) {
  const Grid& g = tree.grid;
  if (static_cast<std::int64_t>(u.size()) != g.total) throw std::invalid_argument("u size does not match grid");
  MomentTable t;
  t.num_moments = g.dim == 1 ? 2 * K + 1 : 1;
  if (K < 0 || (g.dim >= 2 && K != 0)) throw std::invalid_argument("moments support K >= 0 in 1d, K = 0 in 2d/3d");
  std::vector<std::int64_t> sizes;
  std::int64_t tot = 0;
  for (int l = 0; l <= tree.depth; ++l) {
    sizes.push_back(tree.panels_at(l) * t.num_moments);
    tot += sizes.back();
  }
  std::vector<double> flat(tot);
  int64_t adds = 0;
  check(nlg_tree_moments(g.dim, g.n, K, u.data(), flat.data(), &adds));
  if (add_count) *add_count += adds;
  std::int64_t o = 0;
  for (std::int64_t sz : sizes) {
    t.levels.emplace_back(flat.begin() + o, flat.begin() + o + sz);
    o += sz;
  }
  return t;
}

std::int64_t count_recur_calls(const Tree& tree, std::span<const double> radii) {
  if (static_cast<std::int64_t>(radii.size()) != tree.grid.total)
    throw std::invalid_argument("radii size does not match grid");
  int64_t rc = 0, pc = 0;
  check(nlg_tree_count(tree.grid.dim, tree.grid.n, radii.data(), &rc, &pc));
  return rc;
}

namespace {
std::vector<double> node_radii(const KernelSpec& spec, const Grid& grid) {
  std::vector<double> r(grid.total);
  for (std::int64_t i = 0; i < grid.total; ++i) r[i] = spec.horizon_at(node_position(grid, i));
  return r;
}
}  // namespace

const Tree& TruncatedOperator::tree() const {
  if (tree_.grid.total != grid_.total || tree_.grid.dim != grid_.dim) tree_ = build_tree(grid_);
  return tree_;
}

void TruncatedOperator::tree_totals() const {
  if (have_totals_) return;
  const std::vector<double> r = node_radii(spec_, grid_);
  int64_t rc = 0, pc = 0;
  check(nlg_tree_count(grid_.dim, grid_.n, r.data(), &rc, &pc));
  recur_ = rc;
  panels_ = pc;
  have_totals_ = true;
}

const std::vector<Decomposition>& TruncatedOperator::decompositions() const {
  if (decomp_.empty()) {
    const Tree& t = tree();
    decomp_.reserve(grid_.total);
    for (std::int64_t i = 0; i < grid_.total; ++i) {
      const Point x = node_position(grid_, i);
      decomp_.push_back(decompose_region(t, x, spec_.horizon_at(x)));
    }
  }
  return decomp_;
}

std::int64_t TruncatedOperator::recur_calls() const {
  tree_totals();
  return recur_;
}

std::int64_t TruncatedOperator::step2_ops() const {
  const int nm = grid_.dim == 1 ? 2 * spec_.profile.order + 1 : 1;
  std::int64_t per = 0;
  for (int l = 0; l < grid_.levels(); ++l)
    per += (std::int64_t{1} << (grid_.dim * l)) * (std::int64_t{1} << grid_.dim) * nm;
  return applies_ * per;
}

std::int64_t TruncatedOperator::step3_ops() const {
  if (applies_ == 0) return 0;
  tree_totals();
  const int nm = grid_.dim == 1 ? 2 * spec_.profile.order + 1 : 1;
  return applies_ * panels_ * nm;
}

std::vector<double> assemble_dense_matrix(const KernelSpec& spec, const Grid& grid, InclusionRule rule,
                                          ApplyForm form) {
  if (form == ApplyForm::Mass) require_truncated(spec);
  NodeArrays na;
  nlg_desc d = make_desc(spec, grid, na);
  set_profile(d, spec.profile, na);
  if (spec.profile.family == ProfileFamily::PolynomialTruncated) {
    d.route = NLG_ROUTE_TRUNCATED;
    d.rule = rule == InclusionRule::Leaf ? NLG_LEAF : NLG_POINT;
    d.form = form == ApplyForm::Mass ? NLG_MASS : NLG_DIFFERENCE;
    d.divergence = 0;
  } else {
    d.route = NLG_ROUTE_FULL;
    d.rule = NLG_POINT;
    d.form = NLG_DIFFERENCE;
    d.reach = spec.horizon.max_radius();
  }
  PlanGuard g;
  check(nlg_plan_create(&d, &g.p));
  std::vector<double> a(static_cast<std::size_t>(grid.total) * static_cast<std::size_t>(grid.total));
  check(nlg_assemble_dense(g.p, a.data()));
  return a;
}

// ---- Krylov consumer (solve.hpp) -------------------------------------------

namespace {

double norm2(std::span<const double> v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}

double dot(std::span<const double> a, std::span<const double> b) {
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

void check_finite(std::span<const double> v) {
  for (double x : v)
    if (!std::isfinite(x)) throw std::runtime_error("operator produced a non-finite value");
}

}  // namespace

SolveReport solve_dirichlet(const ApplyFn& apply, std::span<const double> f, double tol, std::int64_t max_iter,
                            SolveMethod method, const ApplyFn& apply_transpose) {
  const std::size_t n = f.size();
  SolveReport report;
  report.method = method;
  report.solution.assign(n, 0.0);
  const double fnorm = norm2(f);
  if (fnorm == 0.0) {
    report.converged = true;
    return report;
  }
  if (method == SolveMethod::CGNR && !apply_transpose)
    throw std::invalid_argument("CGNR needs the transpose application");
  std::vector<double>& u = report.solution;
  std::vector<double> r(f.begin(), f.end());
  if (method == SolveMethod::CG) {
    std::vector<double> p = r;
    double rr = dot(r, r);
    for (std::int64_t it = 0; it < max_iter; ++it) {
      if (std::sqrt(rr) / fnorm <= tol) break;
      const std::vector<double> ap = apply(p);
      check_finite(ap);
      const double pap = dot(p, ap);
      if (pap == 0.0) break;
      const double alpha = rr / pap;
      for (std::size_t i = 0; i < n; ++i) {
        u[i] += alpha * p[i];
        r[i] -= alpha * ap[i];
      }
      const double rr_next = dot(r, r);
      const double beta = rr_next / rr;
      rr = rr_next;
      for (std::size_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
      report.iterations = it + 1;
    }
  } else {
    std::vector<double> z = apply_transpose(r);
    std::vector<double> p = z;
    double zz = dot(z, z);
    for (std::int64_t it = 0; it < max_iter; ++it) {
      if (norm2(r) / fnorm <= tol) break;
      const std::vector<double> ap = apply(p);
      check_finite(ap);
      const double denom = dot(ap, ap);
      if (denom == 0.0) break;
      const double alpha = zz / denom;
      for (std::size_t i = 0; i < n; ++i) {
        u[i] += alpha * p[i];
        r[i] -= alpha * ap[i];
      }
      z = apply_transpose(r);
      check_finite(z);
      const double zz_next = dot(z, z);
      const double beta = zz_next / zz;
      zz = zz_next;
      for (std::size_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
      report.iterations = it + 1;
    }
  }
  const std::vector<double> au = apply(u);
  double rn = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    const double d = f[i] - au[i];
    rn += d * d;
  }
  report.final_residual = std::sqrt(rn) / fnorm;
  report.converged = report.final_residual <= tol;
  return report;
}

SolveReport solve_dirichlet(TruncatedOperator& op, std::span<const double> f, double tol, std::int64_t max_iter,
                            SolveMethod method) {
  if (static_cast<std::int64_t>(f.size()) != op.grid().total) throw std::invalid_argument("f size does not match grid");
  SolveReport report;
  report.solution.resize(f.size());
  nlg_solve_report rep{};
  check(nlg_solve_dirichlet(op.native_plan(), f.data(), tol, max_iter,
                            method == SolveMethod::CG ? NLG_SOLVE_CG : NLG_SOLVE_CGNR, report.solution.data(), &rep));
  report.method = method;
  report.iterations = rep.iterations;
  report.final_residual = rep.final_residual;
  report.converged = rep.converged != 0;
  return report;
}

SolveReport solve_dirichlet(TruncatedOperator& op, std::span<const double> f, double tol, std::int64_t max_iter) {
  return solve_dirichlet(op, f, tol, max_iter, choose_method(op.spec()));
}

SolveMethod choose_method(const KernelSpec& spec) {
  const bool symmetric = spec.horizon.kind == HorizonKind::Constant && !spec.coefficient_fn;
  return symmetric ? SolveMethod::CG : SolveMethod::CGNR;
}

std::vector<double> dense_direct_solve(std::span<const double> a_rowmajor, std::span<const double> rhs) {
  const std::size_t n = rhs.size();
  if (a_rowmajor.size() != n * n) throw std::invalid_argument("dense_direct_solve: shape mismatch");
  std::vector<double> a(a_rowmajor.begin(), a_rowmajor.end()), b(rhs.begin(), rhs.end());
  std::vector<std::size_t> piv(n);
  for (std::size_t k = 0; k < n; ++k) {           // partial-pivot LU, in place
    std::size_t p = k;
    for (std::size_t i = k + 1; i < n; ++i)
      if (std::abs(a[i * n + k]) > std::abs(a[p * n + k])) p = i;
    piv[k] = p;
    if (p != k) {
      for (std::size_t j = 0; j < n; ++j) std::swap(a[k * n + j], a[p * n + j]);
      std::swap(b[k], b[p]);
    }
    const double d = a[k * n + k];
    if (d == 0.0) continue;
    for (std::size_t i = k + 1; i < n; ++i) {
      const double l = a[i * n + k] / d;
      a[i * n + k] = l;
      for (std::size_t j = k + 1; j < n; ++j) a[i * n + j] -= l * a[k * n + j];
      b[i] -= l * b[k];
    }
  }
  for (std::size_t k = n; k-- > 0;) {             // back substitution
    double s = b[k];
    for (std::size_t j = k + 1; j < n; ++j) s -= a[k * n + j] * b[j];
    b[k] = s / a[k * n + k];
  }
  return b;
}

std::vector<double> apply_split(const KernelSpec& spec, const Grid& grid, int K, std::span<const double> u,
                                const SplitApplyOptions& options) {
  if (spec.profile.family != ProfileFamily::InverseS)
    throw std::invalid_argument("apply_split expects the InverseS profile");
  if (options.backend != SmoothBackend::Dense)
    throw std::invalid_argument("the HODLR smooth backend is out of scope for the GPU build");
  const SplitKernel sk = split(spec.profile, K);
  std::vector<double> out = apply_smooth_dense(sk, spec, grid, u);
  KernelSpec tspec = spec;
  tspec.profile = RadialProfile::truncated_polynomial(K, spec.profile.c);
  std::vector<double> tpart;
  if (options.truncated == TruncatedPath::FastLeafMass) {
    TruncatedOperator op(tspec, grid);
    tpart = op.apply(u);
  } else {
    tpart = apply_truncated_dense(tspec, grid, InclusionRule::Point, u, ApplyForm::Difference);
  }
  for (std::size_t i = 0; i < out.size(); ++i) out[i] += tpart[i];
  return out;
}

LocalLimitProbe local_limit_probe(const RadialProfile& profile, double delta, const Grid& grid) {
  if (grid.dim != 1) throw std::invalid_argument("local_limit_probe is a 1d diagnostic");
  KernelSpec spec;
  spec.dim = 1;
  spec.profile = profile;
  spec.horizon = {HorizonKind::Constant, delta};
  std::vector<double> u(grid.total);
  for (std::int64_t i = 0; i < grid.total; ++i) {
    const double x = (static_cast<double>(i) + 0.5) * grid.h;
    u[i] = x * x;
  }
  const auto lu = apply_full_dense(spec, grid, u);
  LocalLimitProbe probe;
  for (std::int64_t i = 0; i < grid.total; ++i) {
    const double x = (static_cast<double>(i) + 0.5) * grid.h;
    if (x > delta && 1.0 - x > delta) {
      probe.interior.push_back(i);
      probe.values.push_back(lu[i]);
    }
  }
  return probe;
}

// ---- bench helpers (bench.cpp:10-72) --------------------------------------

std::vector<double> random_vector(std::int64_t n, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  std::vector<double> v(n);
  for (auto& x : v) x = dist(rng);
  return v;
}

double fit_loglog_slope(std::span<const double> x, std::span<const double> y) {
  if (x.size() != y.size() || x.size() < 2) throw std::invalid_argument("slope fit needs matched samples, >= 2");
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  const double n = static_cast<double>(x.size());
  for (std::size_t i = 0; i < x.size(); ++i) {
    const double lx = std::log(x[i]), ly = std::log(y[i]);
    sx += lx;
    sy += ly;
    sxx += lx * lx;
    sxy += lx * ly;
  }
  return (n * sxy - sx * sy) / (n * sxx - sx * sx);
}

BenchRecord run_apply_case(const KernelSpec& spec, const Grid& grid, std::uint64_t seed, int n_vectors) {
  using clk = std::chrono::steady_clock;
  BenchRecord rec;
  rec.N = grid.total;
  TruncatedOperator op(spec, grid);
  for (int v = 0; v < n_vectors; ++v) {
    const auto u = random_vector(grid.total, seed + static_cast<std::uint64_t>(v));
    const auto t0 = clk::now();
    const auto fast = op.apply(u);
    const auto t1 = clk::now();
    std::int64_t pairs = 0;
    const auto dense = apply_truncated_dense(spec, grid, InclusionRule::Leaf, u, ApplyForm::Mass, &pairs);
    const auto t2 = clk::now();
    rec.fast_wall_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    rec.dense_wall_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(t2 - t1).count();
    rec.dense_pairs += pairs;
    double mx = 0.0, md = 0.0;
    for (std::int64_t i = 0; i < grid.total; ++i) {
      mx = std::max(mx, std::abs(dense[i]));
      md = std::max(md, std::abs(fast[i] - dense[i]));
    }
    rec.max_rel_err_vs_dense = std::max(rec.max_rel_err_vs_dense, mx > 0.0 ? md / mx : md);
  }
  // Step-1 instruments, computed on the host by the same Algorithm 1 the
  // reference runs in its constructor (counters match it exactly)
  rec.recur_calls = op.recur_calls();
  rec.step2_ops = op.step2_ops();
  rec.step3_ops = op.step3_ops();
  return rec;
}

}  // namespace nonloc
