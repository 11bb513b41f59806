// paper_1905_08375_b200/csrc/tree.cpp — the reference's Step-1 tree
// instruments (tree.hpp:13-53, tree.cpp:35-58,104-173), host side.
//
// The GPU apply never builds panel lists (row spans replace them, SURVEY §8(a)
// a4); these exist for API parity: decompose_region's panel lists, the
// recursion-call counts the reference reports as its complexity instrument
// (count_recur_calls, TruncatedOperator::recur_calls), the per-node panel
// counts behind step3_ops, and accumulate_moments. Algorithm 1: a dyadic panel
// inside the closed ball is taken whole; a panel meeting the open ball is split
// (or taken whole at leaf level); anything else is dropped. The traversal here
// is an explicit-stack pre-order walk (children in axis-major `which` order), so
// panel lists come out in the reference's order; counting over all nodes runs
// on host threads. Predicates follow geometry.cpp:47-76 operation by operation
// (compiled without FMA contraction).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "plan.hpp"

namespace nlg {
namespace {

struct Cursor {
  int level;
  int64_t k[3];
};

struct Box {
  double lo[3], hi[3];
};

Box cursor_box(int dim, const Cursor& c) {
  const double w = 1.0 / static_cast<double>(int64_t{1} << c.level);
  Box b{};
  for (int j = 0; j < dim; ++j) {
    b.lo[j] = static_cast<double>(c.k[j]) * w;
    b.hi[j] = static_cast<double>(c.k[j] + 1) * w;
  }
  return b;
}

// closed containment: every corner within r (cube_inside_ball)
bool inside(int dim, const Box& b, const double* x, double r) {
  const double r2 = r * r;
  for (int corner = 0; corner < (1 << dim); ++corner) {
    double d2 = 0.0;
    for (int j = 0; j < dim; ++j) {
      const double d = (((corner >> j) & 1) ? b.hi[j] : b.lo[j]) - x[j];
      d2 += d * d;
    }
    if (d2 > r2) return false;
  }
  return true;
}

// open intersection: squared distance to the box below r^2 (cube_intersects_ball)
bool meets(int dim, const Box& b, const double* x, double r) {
  double d2 = 0.0;
  for (int j = 0; j < dim; ++j) {
    double d = 0.0;
    if (b.lo[j] > x[j]) d = b.lo[j] - x[j];
    else if (b.hi[j] < x[j]) d = b.hi[j] - x[j];
    else continue;
    d2 += d * d;
  }
  return d2 < r * r;
}

int64_t flat_index(int dim, const Cursor& c) {
  const int64_t per_axis = int64_t{1} << c.level;
  int64_t f = 0;
  for (int j = 0; j < dim; ++j) f = f * per_axis + c.k[j];
  return f;
}

int depth_of(int64_t n) {
  int l = 0;
  for (int64_t m = n; m > 1; m >>= 1) ++l;
  return l;
}

// Walks Algorithm 1 for one ball; emit(level, index) for every taken panel.
// Returns the number of visited panels (= the reference's recur calls).
template <typename Emit>
int64_t walk(int dim, int depth, const double* x, double r, Emit&& emit) {
  std::vector<Cursor> stack;
  stack.reserve(static_cast<size_t>(depth) * ((1 << dim) - 1) + 2);
  stack.push_back(Cursor{0, {0, 0, 0}});
  int64_t visits = 0;
  while (!stack.empty()) {
    const Cursor c = stack.back();
    stack.pop_back();
    ++visits;
    const Box b = cursor_box(dim, c);
    if (inside(dim, b, x, r)) {
      emit(c.level, flat_index(dim, c));
      continue;
    }
    if (!meets(dim, b, x, r)) continue;
    if (c.level == depth) {
      emit(c.level, flat_index(dim, c));
      continue;
    }
    for (int which = (1 << dim) - 1; which >= 0; --which) {   // reversed push: pre-order pops 0 first
      Cursor ch{c.level + 1, {0, 0, 0}};
      for (int j = 0; j < dim; ++j) ch.k[j] = 2 * c.k[j] + ((which >> j) & 1);
      stack.push_back(ch);
    }
  }
  return visits;
}

void node_position(int dim, int64_t n, int64_t i, double* x) {
  const double h = 1.0 / static_cast<double>(n);
  int64_t rest = i;
  for (int j = dim - 1; j >= 0; --j) {
    x[j] = (static_cast<double>(rest % n) + 0.5) * h;
    rest /= n;
  }
}

}  // namespace

void tree_decompose(int dim, int64_t n, const double* center, double radius, std::vector<int>& levels,
                    std::vector<int64_t>& indices, int64_t& recur_calls) {
  levels.clear();
  indices.clear();
  recur_calls = walk(dim, depth_of(n), center, radius, [&](int l, int64_t f) {
    levels.push_back(l);
    indices.push_back(f);
  });
}

void tree_count(int dim, int64_t n, const double* radii, int64_t& recur_calls, int64_t& panels) {
  int64_t total = 1;
  for (int j = 0; j < dim; ++j) total *= n;
  const int depth = depth_of(n);
  const unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<int64_t> rc(nt, 0), pc(nt, 0);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t) {
    th.emplace_back([&, t] {
      double x[3] = {0, 0, 0};
      for (int64_t i = t; i < total; i += nt) {
        node_position(dim, n, i, x);
        int64_t np = 0;
        rc[t] += walk(dim, depth, x, radii[i], [&](int, int64_t) { ++np; });
        pc[t] += np;
      }
    });
  }
  for (auto& t : th) t.join();
  recur_calls = 0;
  panels = 0;
  for (unsigned t = 0; t < nt; ++t) {
    recur_calls += rc[t];
    panels += pc[t];
  }
}

// Per-panel partial sums M_m(Q) = sum_{x_k in Q} x_k^m u_k, levels 0..L
// flattened level-major; parents are the sums of their 2^d children in child
// order (tree.cpp:115-161). Returns the number of additions.
int64_t tree_moments(int dim, int64_t n, int K, const double* u, double* out) {
  const int depth = depth_of(n);
  const int nm = dim == 1 ? 2 * K + 1 : 1;
  std::vector<int64_t> off(depth + 2, 0);
  for (int l = 0; l <= depth; ++l) off[l + 1] = off[l] + (int64_t{1} << (dim * l)) * nm;
  std::fill(out, out + off[depth + 1], 0.0);
  int64_t total = 1;
  for (int j = 0; j < dim; ++j) total *= n;
  double* leaves = out + off[depth];
  const double h = 1.0 / static_cast<double>(n);
  for (int64_t i = 0; i < total; ++i) {
    if (dim == 1) {
      const double x = (static_cast<double>(i % n) + 0.5) * h;
      double v = u[i];
      for (int m = 0; m < nm; ++m) {
        leaves[i * nm + m] = v;
        v *= x;
      }
    } else {
      leaves[i] = u[i];
    }
  }
  int64_t adds = 0;
  const int nchild = 1 << dim;
  for (int l = depth - 1; l >= 0; --l) {
    const int64_t per_axis = int64_t{1} << l;
    const int64_t count = int64_t{1} << (dim * l);
    double* cur = out + off[l];
    const double* fine = out + off[l + 1];
    for (int64_t p = 0; p < count; ++p) {
      int64_t k[3] = {0, 0, 0}, rest = p;
      for (int j = dim - 1; j >= 0; --j) {
        k[j] = rest % per_axis;
        rest /= per_axis;
      }
      for (int which = 0; which < nchild; ++which) {
        int64_t f = 0;
        for (int j = 0; j < dim; ++j) f = f * (2 * per_axis) + (2 * k[j] + ((which >> j) & 1));
        for (int m = 0; m < nm; ++m) {
          cur[p * nm + m] += fine[f * nm + m];
          ++adds;
        }
      }
    }
  }
  return adds;
}

}  // namespace nlg
