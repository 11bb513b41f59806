// paper_1905_08375_b200/csrc/plan.cu — the C-ABI (include/nlgpu.h).
//
// nlg_plan_create is Step 1 of the reference (TruncatedOperator ctor,
// operators.cpp:102-124): it validates the spec, uploads the per-node delta /
// C / kappa arrays the reference caches (delta_, coeff_, operators.cpp:119-120)
// and prepares the fast method. There is no panel list: the GPU replaces
// Algorithm 1 by spans / scans computed on the fly.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include "plan.hpp"

struct nlg_plan {
  nlg::Plan p;
};

namespace nlg {
namespace {

thread_local std::string g_last_error;

nlg_status fail(nlg_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <typename F>
nlg_status guard(F&& f) {
  try {
    g_last_error.clear();
    f();
    return NLG_OK;
  } catch (const Error& e) {
    return fail(e.code, e.msg);
  } catch (const std::bad_alloc&) {
    return fail(NLG_ERUNTIME, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(NLG_ERUNTIME, e.what());
  }
}

void require(bool ok, const char* msg, nlg_status code = NLG_EINVAL) {
  if (!ok) throw Error{code, msg};
}

int64_t ipow(int64_t n, int d) {
  int64_t r = 1;
  for (int j = 0; j < d; ++j) r *= n;
  return r;
}

// Window radius (cells) of a node with horizon `radius`: the direct kernel
// walks +-(floor(radius/h) + 2), a superset of window_around (operators.cpp:31-42).
int64_t window_cells(double radius, double h) {
  return static_cast<int64_t>(std::floor(radius / h)) + 2;
}

double desc_radius(const nlg_desc& d, double delta_max) {
  double r = delta_max;
  if (d.family <= 3 && d.route == NLG_ROUTE_FULL && d.reach > 0) r = std::max(r, d.reach);
  return r;
}

void validate(const nlg_desc& d) {
  require(d.dim >= 1 && d.dim <= 3, "grid dimension must be 1, 2 or 3");
  require(d.n >= 2, "grid n must be >= 2");
  require(d.family >= 0 && d.family <= 5, "unknown kernel family");
  require(d.route >= 0 && d.route <= 2, "unknown route");
  require(d.rule == 0 || d.rule == 1, "unknown inclusion rule");
  require(d.form == 0 || d.form == 1, "unknown apply form");
  require(d.exterior == 0 || d.exterior == 1, "unknown exterior mode");
  if (d.family == NLG_TRUNCATED || d.family == NLG_KAPPA) {
    require(d.poly && d.npoly >= 1 && d.npoly <= kMaxPoly, "polynomial coefficients required");
  }
  if (d.family == NLG_KAPPA) require(d.tail && d.ntail >= 1 && d.ntail <= kMaxTail, "kappa tail required");
  if (d.family == NLG_TRUNCATED && d.route != NLG_ROUTE_TRUNCATED && d.route != NLG_ROUTE_FULL)
    throw Error{NLG_EINVAL, "truncated profile: route must be TRUNCATED or FULL"};
  if (d.family == NLG_FRACTIONAL || d.family == NLG_PERIDYNAMIC)
    require(d.rule == NLG_POINT && d.form == NLG_DIFFERENCE,
            "fractional / peridynamic kernels use the Point rule, Difference form");
  if (d.route == NLG_ROUTE_TRUNCATED && d.family <= 3)
    require(d.family == NLG_TRUNCATED, "operation requires a PolynomialTruncated profile");
  const int64_t rb = d.row_begin, re = d.row_end == 0 ? d.n : d.row_end;
  require(rb >= 0 && rb < re && re <= d.n, "invalid slab rows");
}

}  // namespace

static cudaEvent_t take_event(Plan& P) {
  if (!P.sprof.pool.empty()) {
    cudaEvent_t e = P.sprof.pool.back();
    P.sprof.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  NLG_CUDA(cudaEventCreate(&e));
  return e;
}

void stage_begin(Plan& P, cudaStream_t s, int stage, cudaEvent_t* ev) {
  (void)stage;
  *ev = nullptr;
  if (!P.sprof.on) return;
  *ev = take_event(P);
  NLG_CUDA(cudaEventRecord(*ev, s));
}

void stage_end(Plan& P, cudaStream_t s, int stage, cudaEvent_t ev, int nlaunch) {
  P.launches += nlaunch;
  P.sprof.launches[stage] += nlaunch;
  if (!P.sprof.on || !ev) return;
  cudaEvent_t e2 = take_event(P);
  NLG_CUDA(cudaEventRecord(e2, s));
  P.sprof.pending.push_back({stage, ev, e2});
}

}  // namespace nlg

using namespace nlg;

extern "C" {

const char* nlg_last_error(void) { return g_last_error.c_str(); }
int nlg_abi_version(void) { return NLG_ABI_VERSION; }

nlg_status nlg_halo_rows(const nlg_desc* desc, double delta_max, int64_t* halo) {
  return guard([&] {
    require(desc && halo, "null argument");
    validate(*desc);
    const double h = 1.0 / static_cast<double>(desc->n);
    const double dm = std::max(std::max(delta_max, desc->delta0), desc->reach);
    *halo = window_cells(desc_radius(*desc, dm), h);
  });
}

nlg_status nlg_plan_create(const nlg_desc* desc, nlg_plan** out) {
  nlg_plan* plan = nullptr;
  nlg_status st = guard([&] {
    require(desc && out, "null argument");
    const nlg_desc& d = *desc;
    validate(d);
    plan = new nlg_plan();
    Plan& P = plan->p;
    P.family = d.family;
    P.route = d.route;
    P.rule = d.rule;
    P.form = d.form;
    P.exterior = d.exterior;
    P.divergence = d.divergence;
    P.device = d.device;
    P.delta0 = d.delta0;
    P.coeff0 = d.coeff0;
    P.reach = d.reach;
    Profile& pr = P.prof;
    std::memset(&pr, 0, sizeof(pr));
    pr.family = d.family;
    pr.route = d.route;
    pr.npoly = d.poly ? d.npoly : 0;
    pr.ntail = d.tail ? d.ntail : 0;
    pr.order = d.order;
    pr.c = d.c;
    pr.alpha = d.alpha;
    for (int j = 0; j < pr.npoly; ++j) pr.poly[j] = d.poly[j];
    for (int j = 0; j < pr.ntail; ++j) pr.tail[j] = d.tail[j];

    Geom& g = P.geom;
    g.dim = d.dim;
    g.n = d.n;
    g.h = 1.0 / static_cast<double>(d.n);
    g.hd = g.h;
    for (int j = 1; j < d.dim; ++j) g.hd *= g.h;
    g.stride0 = ipow(d.n, d.dim - 1);
    g.row_begin = d.row_begin;
    g.row_end = d.row_end == 0 ? d.n : d.row_end;

    // Halo rows: sharded plans (row range != whole grid) read their input
    // rows [rb - H, re + H); H comes from the global horizon bound, which the
    // caller states in `reach` when delta is an array (nlg_halo_rows gives the
    // same H, so the caller can size its arrays first).
    const bool sharded = !(g.row_begin == 0 && g.row_end == d.n);
    if (sharded && d.delta) require(d.reach > 0.0, "sharded plan with a delta array needs reach = max delta");
    const int64_t halo = window_cells(desc_radius(d, std::max(d.delta0, d.reach)), g.h);
    {
      const int64_t lo = std::min<int64_t>(halo, g.row_begin);
      const int64_t hi = std::min<int64_t>(halo, d.n - g.row_end);
      const int64_t cnt = (g.row_end + hi - (g.row_begin - lo)) * g.stride0;
      double dm = d.delta0;
      if (d.delta)
        for (int64_t i = 0; i < cnt; ++i) dm = std::max(dm, d.delta[i]);
      P.delta_max = dm;
      if (sharded && d.delta) require(dm <= d.reach, "reach must bound every delta");
    }
    require(P.delta_max > 0.0, "radius must be positive");
    // nlgpu.h: reach <= 0 means the max delta. With the divergence horizon
    // (delta_x + delta_y)/2 can exceed delta_x, so the window must use it.
    if (P.reach <= 0.0 && P.divergence) P.reach = P.delta_max;
    P.halo_lo = std::min<int64_t>(halo, g.row_begin);
    P.halo_hi = std::min<int64_t>(halo, d.n - g.row_end);
    g.in_begin = g.row_begin - P.halo_lo;
    g.in_end = g.row_end + P.halo_hi;
    P.n_in = (g.in_end - g.in_begin) * g.stride0;
    P.n_out = (g.row_end - g.row_begin) * g.stride0;

    NLG_CUDA(cudaSetDevice(P.device));
    NLG_CUDA(cudaStreamCreateWithFlags(&P.stream, cudaStreamNonBlocking));
    const size_t bytes_in = sizeof(double) * static_cast<size_t>(P.n_in);
    if (d.delta) {
      NLG_CUDA(cudaMalloc(&P.d_delta, bytes_in));
      NLG_CUDA(cudaMemcpyAsync(P.d_delta, d.delta, bytes_in, cudaMemcpyHostToDevice, P.stream));
    }
    if (d.coeff) {
      NLG_CUDA(cudaMalloc(&P.d_coeff, bytes_in));
      NLG_CUDA(cudaMemcpyAsync(P.d_coeff, d.coeff, bytes_in, cudaMemcpyHostToDevice, P.stream));
    }
    if (d.kappa) {
      NLG_CUDA(cudaMalloc(&P.d_kappa, bytes_in));
      NLG_CUDA(cudaMemcpyAsync(P.d_kappa, d.kappa, bytes_in, cudaMemcpyHostToDevice, P.stream));
    }
    NLG_CUDA(cudaMalloc(&P.d_pairs, sizeof(unsigned long long)));
    direct_frac_setup(P);

    // fast method selection
    if (P.family == NLG_TRUNCATED && P.route == NLG_ROUTE_TRUNCATED && pr.npoly == 1) {
      P.fast_method = 1;
      spans_setup(P);
    } else if (P.family == NLG_TRUNCATED && P.route == NLG_ROUTE_TRUNCATED && g.dim == 1 && pr.npoly <= 4 &&
               P.form == NLG_MASS && !P.divergence) {
      moments_setup(P, pr.npoly - 1);            // 1-D K = 1..3: centred moment scans
    } else if (P.family == NLG_FRACTIONAL && g.dim == 1) {
      expsum_setup(P, d);                       // wide horizons: exponential-sum scans
      if (P.fast_method == 0) stencil_setup(P, d);   // narrow ones: 1-D stencil
    } else if ((P.family == NLG_FRACTIONAL || P.family == NLG_PERIDYNAMIC) && g.dim >= 2) {
      stencil_setup(P, d);
    } else {
      P.fast_method = 0;
    }
    NLG_CUDA(cudaStreamSynchronize(P.stream));
    *out = plan;
  });
  if (st != NLG_OK && plan) {
    nlg_plan_destroy(plan);
  }
  return st;
}

void nlg_plan_destroy(nlg_plan* plan) {
  if (!plan) return;
  Plan& P = plan->p;
  cudaSetDevice(P.device);
  if (P.stream) cudaStreamSynchronize(P.stream);
  for (auto& r : P.sprof.pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : P.sprof.pool) cudaEventDestroy(e);
  spans_free(P);
  expsum_free(P);
  stencil_free(P);
  cudaFree(P.d_delta);
  cudaFree(P.d_coeff);
  cudaFree(P.d_kappa);
  cudaFree(P.d_u);
  cudaFree(P.d_out);
  cudaFree(P.d_pairs);
  cudaFree(P.d_targets);
  cudaFree(P.d_wfrac);
  if (P.stream) cudaStreamDestroy(P.stream);
  if (P.h2d_stream) cudaStreamDestroy(P.h2d_stream);
  if (P.d2h_stream) cudaStreamDestroy(P.d2h_stream);
  for (auto e : P.pipe_ev) cudaEventDestroy(e);
  delete plan;
}

nlg_status nlg_plan_info(const nlg_plan* plan, nlg_info* info) {
  return guard([&] {
    require(plan && info, "null argument");
    const Plan& P = plan->p;
    info->halo_lo = P.halo_lo;
    info->halo_hi = P.halo_hi;
    info->n_in = P.n_in;
    info->n_out = P.n_out;
    info->fast_method = P.fast_method;
    info->exp_terms = P.es.terms;
    info->near_cells = P.es.near;
    info->far_rel_err = P.es.rel_err;
    info->fft_len = 0;
    info->fft_rows = 0;
    if (P.es_state) expsum_fft_info(P, info->fft_len, info->fft_rows);
    if (P.st_state) info->fft_len = stencil_fft_len(P);
  });
}

namespace {

int components(const Plan& P) { return P.family == NLG_PERIDYNAMIC ? P.geom.dim : 1; }

void ensure_staging(Plan& P) {
  const int nc = components(P);
  if (!P.d_u) NLG_CUDA(cudaMalloc(&P.d_u, sizeof(double) * nc * P.n_in));
  if (!P.d_out) NLG_CUDA(cudaMalloc(&P.d_out, sizeof(double) * nc * P.n_out));
}

void fast_dev(Plan& P, const double* u, double* out, cudaStream_t s) {
  switch (P.fast_method) {
    case 1: spans_apply(P, u, out, s); break;
    case 4: moments_apply(P, u, out, s); break;
    case 2: expsum_apply(P, u, out, s); break;
    case 3: {
      if (stencil_box(P)) {   // box FFT mode: its passes and tie pass are stages of their own
        stencil_apply(P, u, out, s);
        break;
      }
      cudaEvent_t ev;
      stage_begin(P, s, kStStencil, &ev);
      stencil_apply(P, u, out, s);
      stage_end(P, s, kStStencil, ev, stencil_launches(P));
      break;
    }
    default: {
      cudaEvent_t ev;
      stage_begin(P, s, kStDirect, &ev);
      launch_direct(P, u, out, nullptr, 0, nullptr, s);
      stage_end(P, s, kStDirect, ev, 1);
      break;
    }
  }
  NLG_CUDA(cudaGetLastError());
  ++P.fast_applies;
}

// The chunked host pipeline of nlg_apply_fast: 2-D / 3-D stencil (scalar and
// peridynamic) and box-FFT plans of at least 4 Mi nodes. Input rows travel H2D in chunks on one
// copy stream; each output row range is computed as soon as every input row
// it reads (H rows either side) is resident, and travels D2H on a second copy
// stream while the next chunks copy in and compute: PCIe in, PCIe out and the
// apply overlap instead of running back to back.
bool pipelinable(const Plan& P) {
  return P.fast_method == 3 && P.geom.dim >= 2 && P.n_out >= (int64_t{1} << 22) && stencil_reach_rows(P) > 0;
}

void apply_fast_pipelined(Plan& P, const double* u, double* out) {
  const Geom& g = P.geom;
  const int64_t st = g.stride0, rows_in = g.in_end - g.in_begin, rows_out = g.row_end - g.row_begin;
  const int64_t H = stencil_reach_rows(P);
  const bool box = stencil_box(P);
  const int nc = components(P);
  static const int env_chunks = [] { const char* e = std::getenv("NLG_PIPE_CHUNKS"); return e ? std::atoi(e) : 0; }();
  const int nch = static_cast<int>(std::min<int64_t>(env_chunks > 0 ? env_chunks : (box ? 24 : 16), rows_in));
  if (!P.h2d_stream) {
    NLG_CUDA(cudaStreamCreateWithFlags(&P.h2d_stream, cudaStreamNonBlocking));
    NLG_CUDA(cudaStreamCreateWithFlags(&P.d2h_stream, cudaStreamNonBlocking));
  }
  while (static_cast<int>(P.pipe_ev.size()) < 2 * nch) {
    cudaEvent_t e;
    NLG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    P.pipe_ev.push_back(e);
  }
  int64_t q_done = 0;
  for (int k = 0; k < nch; ++k) {
    const int64_t i0 = rows_in * k / nch, i1 = rows_in * (k + 1) / nch;
    for (int c = 0; c < nc; ++c)   // (peridynamics: one row chunk per component plane)
      NLG_CUDA(cudaMemcpyAsync(P.d_u + c * P.n_in + i0 * st, u + c * P.n_in + i0 * st, sizeof(double) * (i1 - i0) * st,
                               cudaMemcpyHostToDevice, P.h2d_stream));
    NLG_CUDA(cudaEventRecord(P.pipe_ev[k], P.h2d_stream));
    NLG_CUDA(cudaStreamWaitEvent(P.stream, P.pipe_ev[k], 0));
    if (box) stencil_box_in(P, P.d_u, i0, i1, P.stream);
    // output rows whose whole window [r - H, r + H] is resident
    const int64_t tile = box ? 1 : stencil_row_tile(P);
    const int64_t q_ready =
        k == nch - 1 ? rows_out
                     : std::clamp<int64_t>(g.in_begin + i1 - H - g.row_begin, 0, rows_out) / tile * tile;
    if (q_ready <= q_done) continue;
    if (box) {
      stencil_box_out(P, P.d_u, P.d_out, q_done, q_ready, P.stream);
    } else {
      cudaEvent_t ev;
      stage_begin(P, P.stream, kStStencil, &ev);
      stencil_apply_rows(P, P.d_u, P.d_out, q_done, q_ready, P.stream);
      stage_end(P, P.stream, kStStencil, ev, 1);
    }
    NLG_CUDA(cudaGetLastError());
    NLG_CUDA(cudaEventRecord(P.pipe_ev[nch + k], P.stream));
    NLG_CUDA(cudaStreamWaitEvent(P.d2h_stream, P.pipe_ev[nch + k], 0));
    for (int c = 0; c < nc; ++c)
      NLG_CUDA(cudaMemcpyAsync(out + c * P.n_out + q_done * st, P.d_out + c * P.n_out + q_done * st,
                               sizeof(double) * (q_ready - q_done) * st, cudaMemcpyDeviceToHost, P.d2h_stream));
    q_done = q_ready;
  }
  NLG_CUDA(cudaStreamSynchronize(P.d2h_stream));
  NLG_CUDA(cudaStreamSynchronize(P.stream));
  ++P.fast_applies;
}

}  // namespace

nlg_status nlg_apply_fast(nlg_plan* plan, const double* u, double* out) {
  return guard([&] {
    require(plan && u && out, "null argument");
    Plan& P = plan->p;
    NLG_CUDA(cudaSetDevice(P.device));
    ensure_staging(P);
    if (pipelinable(P) && !std::getenv("NLG_NO_PIPELINE")) {
      apply_fast_pipelined(P, u, out);
      return;
    }
    const int nc = components(P);
    NLG_CUDA(cudaMemcpyAsync(P.d_u, u, sizeof(double) * nc * P.n_in, cudaMemcpyHostToDevice, P.stream));
    fast_dev(P, P.d_u, P.d_out, P.stream);
    NLG_CUDA(cudaMemcpyAsync(out, P.d_out, sizeof(double) * nc * P.n_out, cudaMemcpyDeviceToHost, P.stream));
    NLG_CUDA(cudaStreamSynchronize(P.stream));
  });
}

// Split-phase device apply for sharded plans: _begin enqueues the work that
// does not read u's halo rows (box FFT: the x / y transforms of the owned
// planes), so a caller can exchange the halos meanwhile; _end the rest. For
// every other method _begin does nothing and _end is nlg_apply_fast_dev.
nlg_status nlg_apply_fast_dev_begin(nlg_plan* plan, const double* u_dev, double* out_dev, void* stream) {
  return guard([&] {
    require(plan && u_dev && out_dev, "null argument");
    Plan& P = plan->p;
    NLG_CUDA(cudaSetDevice(P.device));
    P.split_begun = false;
    P.split_lo = P.split_hi = 0;
    if (P.fast_method == 3 && stencil_box(P)) {
      const int64_t rows_in = P.geom.in_end - P.geom.in_begin;
      stencil_box_in(P, u_dev, P.halo_lo, rows_in - P.halo_hi, static_cast<cudaStream_t>(stream));
      NLG_CUDA(cudaGetLastError());
      P.split_begun = true;
    } else if (P.fast_method == 3 && P.geom.dim >= 2 && (P.halo_lo > 0 || P.halo_hi > 0)) {
      // stencil slab: the output rows whose whole window lies in the owned
      // input rows (r >= H past a lower halo, r < rows_out - H before an upper
      // one), cut at CTA-row multiples so the result is bit-identical
      const int64_t rows_out = P.geom.row_end - P.geom.row_begin, H = stencil_reach_rows(P);
      const int64_t tile = stencil_row_tile(P);
      const int64_t lo = P.halo_lo > 0 ? (H + tile - 1) / tile * tile : 0;
      const int64_t hi = P.halo_hi > 0 ? (rows_out - H) / tile * tile : rows_out;
      if (hi > lo) {
        cudaEvent_t ev;
        stage_begin(P, static_cast<cudaStream_t>(stream), kStStencil, &ev);
        stencil_apply_rows(P, u_dev, out_dev, lo, hi, static_cast<cudaStream_t>(stream));
        stage_end(P, static_cast<cudaStream_t>(stream), kStStencil, ev, 1);
        NLG_CUDA(cudaGetLastError());
        P.split_lo = lo;
        P.split_hi = hi;
        P.split_begun = true;
      }
    }
  });
}

nlg_status nlg_apply_fast_dev_end(nlg_plan* plan, const double* u_dev, double* out_dev, void* stream) {
  return guard([&] {
    require(plan && u_dev && out_dev, "null argument");
    Plan& P = plan->p;
    NLG_CUDA(cudaSetDevice(P.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (P.split_begun && stencil_box(P)) {
      const int64_t rows_in = P.geom.in_end - P.geom.in_begin;
      stencil_box_in(P, u_dev, 0, P.halo_lo, s);
      stencil_box_in(P, u_dev, rows_in - P.halo_hi, rows_in, s);
      stencil_box_out(P, u_dev, out_dev, 0, P.geom.row_end - P.geom.row_begin, s);
      NLG_CUDA(cudaGetLastError());
      ++P.fast_applies;
      P.split_begun = false;
      return;
    }
    if (P.split_begun) {   // stencil slab: the edge rows that read the halos
      const int64_t rows_out = P.geom.row_end - P.geom.row_begin;
      cudaEvent_t ev;
      stage_begin(P, s, kStStencil, &ev);
      stencil_apply_rows(P, u_dev, out_dev, 0, P.split_lo, s);
      stencil_apply_rows(P, u_dev, out_dev, P.split_hi, rows_out, s);
      stage_end(P, s, kStStencil, ev, (P.split_lo > 0) + (P.split_hi < rows_out));
      NLG_CUDA(cudaGetLastError());
      ++P.fast_applies;
      P.split_begun = false;
      return;
    }
    fast_dev(P, u_dev, out_dev, s);
  });
}

nlg_status nlg_apply_fast_dev(nlg_plan* plan, const double* u_dev, double* out_dev, void* stream) {
  return guard([&] {
    require(plan && u_dev && out_dev, "null argument");
    Plan& P = plan->p;
    NLG_CUDA(cudaSetDevice(P.device));
    fast_dev(P, u_dev, out_dev, static_cast<cudaStream_t>(stream));
  });
}

nlg_status nlg_apply_direct(nlg_plan* plan, const double* u, double* out, int64_t* pair_count) {
  return guard([&] {
    require(plan && u && out, "null argument");
    Plan& P = plan->p;
    NLG_CUDA(cudaSetDevice(P.device));
    ensure_staging(P);
    const int nc = components(P);
    NLG_CUDA(cudaMemcpyAsync(P.d_u, u, sizeof(double) * nc * P.n_in, cudaMemcpyHostToDevice, P.stream));
    NLG_CUDA(cudaMemsetAsync(P.d_pairs, 0, sizeof(unsigned long long), P.stream));
    cudaEvent_t ev;
    stage_begin(P, P.stream, kStDirect, &ev);
    launch_direct(P, P.d_u, P.d_out, nullptr, 0, P.d_pairs, P.stream);
    stage_end(P, P.stream, kStDirect, ev, 1);
    NLG_CUDA(cudaGetLastError());
    unsigned long long pairs = 0;
    NLG_CUDA(cudaMemcpyAsync(out, P.d_out, sizeof(double) * nc * P.n_out, cudaMemcpyDeviceToHost, P.stream));
    NLG_CUDA(cudaMemcpyAsync(&pairs, P.d_pairs, sizeof(pairs), cudaMemcpyDeviceToHost, P.stream));
    NLG_CUDA(cudaStreamSynchronize(P.stream));
    P.last_pairs = static_cast<int64_t>(pairs);
    if (pair_count) *pair_count += P.last_pairs;
  });
}

nlg_status nlg_apply_direct_dev(nlg_plan* plan, const double* u_dev, double* out_dev,
                                int64_t* pair_count_dev, void* stream) {
  return guard([&] {
    require(plan && u_dev && out_dev, "null argument");
    Plan& P = plan->p;
    NLG_CUDA(cudaSetDevice(P.device));
    cudaEvent_t ev;
    stage_begin(P, static_cast<cudaStream_t>(stream), kStDirect, &ev);
    launch_direct(P, u_dev, out_dev, nullptr, 0,
                  reinterpret_cast<unsigned long long*>(pair_count_dev),
                  static_cast<cudaStream_t>(stream));
    stage_end(P, static_cast<cudaStream_t>(stream), kStDirect, ev, 1);
    NLG_CUDA(cudaGetLastError());
  });
}

nlg_status nlg_apply_direct_at(nlg_plan* plan, const double* u, const int64_t* targets,
                               int64_t ntargets, double* out, int64_t* pair_count) {
  return guard([&] {
    require(plan && u && targets && out && ntargets >= 0, "null argument");
    Plan& P = plan->p;
    for (int64_t t = 0; t < ntargets; ++t)
      if (targets[t] < 0 || targets[t] >= P.n_out) throw Error{NLG_ERANGE, "node index out of range"};
    NLG_CUDA(cudaSetDevice(P.device));
    ensure_staging(P);
    if (P.targets_cap < ntargets) {
      cudaFree(P.d_targets);
      P.d_targets = nullptr;
      NLG_CUDA(cudaMalloc(&P.d_targets, sizeof(int64_t) * std::max<int64_t>(ntargets, 1)));
      P.targets_cap = ntargets;
    }
    const int nc = components(P);
    double* d_o = nullptr;
    NLG_CUDA(cudaMalloc(&d_o, sizeof(double) * nc * std::max<int64_t>(ntargets, 1)));
    NLG_CUDA(cudaMemcpyAsync(P.d_u, u, sizeof(double) * nc * P.n_in, cudaMemcpyHostToDevice, P.stream));
    NLG_CUDA(cudaMemcpyAsync(P.d_targets, targets, sizeof(int64_t) * ntargets, cudaMemcpyHostToDevice, P.stream));
    NLG_CUDA(cudaMemsetAsync(P.d_pairs, 0, sizeof(unsigned long long), P.stream));
    launch_direct(P, P.d_u, d_o, P.d_targets, ntargets, P.d_pairs, P.stream);
    unsigned long long pairs = 0;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out, d_o, sizeof(double) * nc * ntargets, cudaMemcpyDeviceToHost, P.stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&pairs, P.d_pairs, sizeof(pairs), cudaMemcpyDeviceToHost, P.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(P.stream);
    cudaFree(d_o);
    if (e != cudaSuccess) throw Error{NLG_ECUDA, cudaGetErrorString(e)};
    if (pair_count) *pair_count = static_cast<int64_t>(pairs);
  });
}

nlg_status nlg_counters(const nlg_plan* plan, int64_t* pairs, int64_t* fast_applies) {
  return guard([&] {
    require(plan, "null argument");
    if (pairs) *pairs = plan->p.last_pairs;
    if (fast_applies) *fast_applies = plan->p.fast_applies;
  });
}

nlg_status nlg_set_profiling(nlg_plan* plan, int on) {
  return guard([&] {
    require(plan, "null argument");
    plan->p.sprof.on = on != 0;
  });
}

static_assert(nlg::kNumStages == NLG_NUM_STAGES, "stage slots of the C-ABI");

nlg_status nlg_stage_times(nlg_plan* plan, double* ms, int64_t* launches, int* nstages) {
  return guard([&] {
    require(plan && ms && launches && nstages, "null argument");
    Plan& P = plan->p;
    NLG_CUDA(cudaSetDevice(P.device));
    for (auto& r : P.sprof.pending) {
      NLG_CUDA(cudaEventSynchronize(r.b));
      float t = 0.f;
      NLG_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
      P.sprof.ms[r.stage] += t;
      P.sprof.pool.push_back(r.a);
      P.sprof.pool.push_back(r.b);
    }
    P.sprof.pending.clear();
    for (int k = 0; k < kNumStages; ++k) {
      ms[k] = P.sprof.ms[k];
      launches[k] = P.sprof.launches[k];
      P.sprof.ms[k] = 0.0;
      P.sprof.launches[k] = 0;
    }
    *nstages = kNumStages;
  });
}

nlg_status nlg_launch_count(const nlg_plan* plan, int64_t* launches) {
  return guard([&] {
    require(plan && launches, "null argument");
    *launches = plan->p.launches;
  });
}

nlg_status nlg_match_polynomial(int K, double c, double* coeffs) {
  return guard([&] {
    require(coeffs, "null argument");
    const auto p = match_polynomial(K, c);
    for (size_t j = 0; j < p.size(); ++j) coeffs[j] = p[j];
  });
}

nlg_status nlg_match_polynomial_exact(int K, int64_t* num, int64_t* den) {
  return guard([&] {
    require(num && den, "null argument");
    require(K >= 0 && K <= 6, "matching order must be in [0, 6]");
    match_polynomial_exact(K, num, den);
  });
}

nlg_status nlg_split(int K, double c, double* poly, double* tail, int* ntail) {
  return guard([&] {
    require(poly && tail && ntail, "null argument");
    std::vector<double> p, t;
    split_kernel(K, c, p, t);
    for (size_t j = 0; j < p.size(); ++j) poly[j] = p[j];
    for (size_t j = 0; j < t.size(); ++j) tail[j] = t[j];
    *ntail = static_cast<int>(t.size());
  });
}

nlg_status nlg_expsum_fit(double alpha, int near, int64_t dmax, double* rate, double* weight,
                          int* terms, double* rel_err) {
  return guard([&] {
    require(rate && weight && terms && rel_err, "null argument");
    require(alpha > 0 && near >= 1 && dmax > near, "invalid exponential-sum window");
    const ExpSum es = fit_exponential_sum(alpha, near, dmax, 0.0);
    require(es.terms <= 64, "too many exponential terms", NLG_ERUNTIME);
    for (int m = 0; m < es.terms; ++m) {
      rate[m] = es.rate[m];
      weight[m] = es.weight[m];
    }
    *terms = es.terms;
    *rel_err = es.rel_err;
  });
}

}  // extern "C"

// ---- matrix view and Krylov consumer ----------------------------------------

namespace nlg {
namespace {

void require_matrix_view(const Plan& P) {
  require(direct_kind(P) <= 3, "matrix view needs a scalar operator (not peridynamic)");
}

}  // namespace
}  // namespace nlg

nlg_status nlg_apply_transpose(nlg_plan* plan, const double* v, double* out) {
  using namespace nlg;
  return guard([&] {
    require(plan && v && out, "null argument");
    Plan& P = plan->p;
    require_matrix_view(P);
    NLG_CUDA(cudaSetDevice(P.device));
    ensure_staging(P);
    NLG_CUDA(cudaMemcpyAsync(P.d_u, v, sizeof(double) * P.n_in, cudaMemcpyHostToDevice, P.stream));
    launch_transpose(P, P.d_u, P.d_out, P.stream);
    NLG_CUDA(cudaGetLastError());
    ++P.launches;
    NLG_CUDA(cudaMemcpyAsync(out, P.d_out, sizeof(double) * P.n_out, cudaMemcpyDeviceToHost, P.stream));
    NLG_CUDA(cudaStreamSynchronize(P.stream));
  });
}

nlg_status nlg_apply_transpose_dev(nlg_plan* plan, const double* v_dev, double* out_dev, void* stream) {
  using namespace nlg;
  return guard([&] {
    require(plan && v_dev && out_dev, "null argument");
    Plan& P = plan->p;
    require_matrix_view(P);
    NLG_CUDA(cudaSetDevice(P.device));
    launch_transpose(P, v_dev, out_dev, static_cast<cudaStream_t>(stream));
    NLG_CUDA(cudaGetLastError());
    ++P.launches;
  });
}

nlg_status nlg_assemble_dense(nlg_plan* plan, double* a) {
  using namespace nlg;
  return guard([&] {
    require(plan && a, "null argument");
    Plan& P = plan->p;
    require_matrix_view(P);
    require(P.n_in == P.n_out, "dense assembly needs an unsharded plan");
    const int64_t N = P.n_out;
    require(N <= 32768, "dense assembly limited to N <= 32768 (N^2 doubles)");
    NLG_CUDA(cudaSetDevice(P.device));
    double* d = nullptr;
    const size_t bytes = sizeof(double) * static_cast<size_t>(N) * static_cast<size_t>(N);
    NLG_CUDA(cudaMalloc(&d, bytes));
    cudaError_t e = cudaMemsetAsync(d, 0, bytes, P.stream);
    if (e == cudaSuccess) {
      launch_assemble(P, d, N, P.stream);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(a, d, bytes, cudaMemcpyDeviceToHost, P.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(P.stream);
    cudaFree(d);
    ++P.launches;
    NLG_CUDA(e);
  });
}

nlg_status nlg_solve_dirichlet(nlg_plan* plan, const double* f, double tol, int64_t max_iter, int method,
                               double* u_out, nlg_solve_report* rep) {
  using namespace nlg;
  std::vector<void*> bufs;
  nlg_status st = guard([&] {
    require(plan && f && u_out && rep, "null argument");
    Plan& P = plan->p;
    require(components(P) == 1, "the solver needs a scalar operator");
    require(P.n_in == P.n_out, "the device solver needs an unsharded plan");
    const int m = method & 0xF;
    const bool direct = (method & NLG_SOLVE_DIRECT) != 0;
    require(m == NLG_SOLVE_CG || m == NLG_SOLVE_CGNR, "unknown solve method");
    if (m == NLG_SOLVE_CGNR) require_matrix_view(P);
    NLG_CUDA(cudaSetDevice(P.device));
    const int64_t n = P.n_out;
    cudaStream_t s = P.stream;
    auto dalloc = [&](size_t count) {
      void* q = nullptr;
      NLG_CUDA(cudaMalloc(&q, count));
      bufs.push_back(q);
      return q;
    };
    const size_t vb = sizeof(double) * static_cast<size_t>(n);
    double* df = static_cast<double*>(dalloc(vb));
    double* du = static_cast<double*>(dalloc(vb));
    double* dr = static_cast<double*>(dalloc(vb));
    double* dp = static_cast<double*>(dalloc(vb));
    double* dap = static_cast<double*>(dalloc(vb));
    double* dz = m == NLG_SOLVE_CGNR ? static_cast<double*>(dalloc(vb)) : nullptr;
    double* scratch = static_cast<double*>(dalloc(sizeof(double) * dot_scratch_doubles()));
    int* bad = static_cast<int*>(dalloc(sizeof(int)));
    NLG_CUDA(cudaMemcpyAsync(df, f, vb, cudaMemcpyHostToDevice, s));
    NLG_CUDA(cudaMemsetAsync(du, 0, vb, s));
    NLG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    // A = -L
    auto applyA = [&](const double* x, double* y) {
      if (direct) launch_direct(P, x, y, nullptr, 0, nullptr, s);
      else fast_dev(P, x, y, s);
      dev_negate(y, n, s);
      NLG_CUDA(cudaGetLastError());
    };
    auto applyAT = [&](const double* x, double* y) {
      launch_transpose(P, x, y, s);
      dev_negate(y, n, s);
      NLG_CUDA(cudaGetLastError());
    };
    auto dot = [&](const double* a, const double* b, const double* chk) {
      dev_dot(a, b, chk, n, scratch, bad, s);
      double v = 0.0;
      int flag = 0;
      NLG_CUDA(cudaMemcpyAsync(&v, scratch + dot_scratch_doubles() - 1, sizeof(double), cudaMemcpyDeviceToHost, s));
      NLG_CUDA(cudaMemcpyAsync(&flag, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
      NLG_CUDA(cudaStreamSynchronize(s));
      if (flag) throw Error{NLG_ERUNTIME, "operator produced a non-finite value"};
      return v;
    };
    *rep = nlg_solve_report{m, 0, 0, 0.0};
    const double fnorm = std::sqrt(dot(df, df, nullptr));
    if (fnorm == 0.0) {
      rep->converged = 1;
      std::memset(u_out, 0, vb);
      return;
    }
    NLG_CUDA(cudaMemcpyAsync(dr, df, vb, cudaMemcpyDeviceToDevice, s));   // r = f - A 0
    if (m == NLG_SOLVE_CG) {
      NLG_CUDA(cudaMemcpyAsync(dp, dr, vb, cudaMemcpyDeviceToDevice, s));
      double rr = dot(dr, dr, nullptr);
      for (int64_t it = 0; it < max_iter; ++it) {
        if (std::sqrt(rr) / fnorm <= tol) break;
        applyA(dp, dap);
        const double pap = dot(dp, dap, dap);
        if (pap == 0.0) break;
        const double alpha = rr / pap;
        dev_axpy2(du, dr, dp, dap, alpha, n, s);
        const double rr_next = dot(dr, dr, nullptr);
        const double beta = rr_next / rr;
        rr = rr_next;
        dev_xpby(dp, dr, beta, n, s);
        rep->iterations = it + 1;
      }
    } else {
      // CG on A^T A u = A^T f; r tracks f - A u
      applyAT(dr, dz);
      NLG_CUDA(cudaMemcpyAsync(dp, dz, vb, cudaMemcpyDeviceToDevice, s));
      double zz = dot(dz, dz, nullptr);
      for (int64_t it = 0; it < max_iter; ++it) {
        if (std::sqrt(dot(dr, dr, nullptr)) / fnorm <= tol) break;
        applyA(dp, dap);
        const double denom = dot(dap, dap, dap);
        if (denom == 0.0) break;
        const double alpha = zz / denom;
        dev_axpy2(du, dr, dp, dap, alpha, n, s);
        applyAT(dr, dz);
        const double zz_next = dot(dz, dz, dz);
        const double beta = zz_next / zz;
        zz = zz_next;
        dev_xpby(dp, dz, beta, n, s);
        rep->iterations = it + 1;
      }
    }
    // the true residual, not the recurrence
    applyA(du, dap);
    dev_diff(dr, df, dap, n, s);
    rep->final_residual = std::sqrt(dot(dr, dr, nullptr)) / fnorm;
    rep->converged = rep->final_residual <= tol;
    NLG_CUDA(cudaMemcpyAsync(u_out, du, vb, cudaMemcpyDeviceToHost, s));
    NLG_CUDA(cudaStreamSynchronize(s));
  });
  for (void* q : bufs) cudaFree(q);
  return st;
}

// ---- Step-1 tree instruments -------------------------------------------------

namespace {
bool pow2(int64_t n) { return n >= 2 && (n & (n - 1)) == 0; }
}  // namespace

nlg_status nlg_tree_decompose(int dim, int64_t n, const double* center, double radius, int64_t cap, int* levels,
                              int64_t* indices, int64_t* npanels, int64_t* recur_calls) {
  using namespace nlg;
  return guard([&] {
    require(center && npanels && recur_calls, "null argument");
    require(dim >= 1 && dim <= 3, "grid dimension must be 1, 2 or 3");
    require(pow2(n), "tree requires n to be a power of two");
    require(radius > 0.0, "radius must be positive");
    std::vector<int> lv;
    std::vector<int64_t> ix;
    tree_decompose(dim, n, center, radius, lv, ix, *recur_calls);
    *npanels = static_cast<int64_t>(lv.size());
    for (int64_t k = 0; k < *npanels && k < cap; ++k) {
      if (levels) levels[k] = lv[k];
      if (indices) indices[k] = ix[k];
    }
  });
}

nlg_status nlg_tree_count(int dim, int64_t n, const double* radii, int64_t* recur_calls, int64_t* panels) {
  using namespace nlg;
  return guard([&] {
    require(radii && recur_calls && panels, "null argument");
    require(dim >= 1 && dim <= 3, "grid dimension must be 1, 2 or 3");
    require(pow2(n), "tree requires n to be a power of two");
    tree_count(dim, n, radii, *recur_calls, *panels);
  });
}

nlg_status nlg_tree_moments(int dim, int64_t n, int K, const double* u, double* out, int64_t* adds) {
  using namespace nlg;
  return guard([&] {
    require(u && out, "null argument");
    require(dim >= 1 && dim <= 3, "grid dimension must be 1, 2 or 3");
    require(pow2(n), "tree requires n to be a power of two");
    require(K >= 0 && (dim == 1 || K == 0), "moments support K >= 0 in 1d, K = 0 in 2d/3d");
    const int64_t a = tree_moments(dim, n, K, u, out);
    if (adds) *adds = a;
  });
}

nlg_status nlg_expsum_fit_narrow(double alpha, int64_t lo, int64_t hi, double tol, int max_terms, double* rate,
                                 double* weight, int* terms, double* rel_err) {
  using namespace nlg;
  return guard([&] {
    require(rate && weight && terms && rel_err, "null argument");
    require(lo >= 1 && hi >= lo && max_terms >= 2, "invalid window");
    const ExpSum es = fit_exponential_sum_narrow(alpha, lo, hi, tol, max_terms);
    *terms = es.terms;
    *rel_err = es.rel_err;
    for (int k = 0; k < es.terms; ++k) {
      rate[k] = es.rate[k];
      weight[k] = es.weight[k];
    }
  });
}
