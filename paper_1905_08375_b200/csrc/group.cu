// paper_1905_08375_b200/csrc/group.cu — multi-GPU plans inside the C-ABI
// (SURVEY §8(e)): one process drives ndev devices, the grid's axis-0 rows are
// split into slabs (one sharded plan per device, nlg_desc.row_begin/row_end),
// u's halo rows move between neighbouring devices by NCCL point-to-point over
// NVLink (ncclCommInitAll: one communicator per device, single process), and
// the halo-independent part of each slab's apply (nlg_apply_fast_dev_begin)
// runs while the halos are in flight on a separate communication stream.
//
// The halo depth is the reference's window (window_around, operators.cpp:31-42):
// rows [x - delta - h, x + delta + h] around an output row, sized by
// nlg_halo_rows. Outputs are disjoint: no other collective on the data path.
//
// NCCL is loaded at run time (dlopen libnccl.so.2) so the library has no link
// dependency on it; a missing NCCL or a failing call is NLG_ENCCL, and
// ncclCommGetAsyncError is checked after every exchange. When a device ordinal
// repeats in the list (one GPU standing in for several slabs: tests, debugging)
// NCCL cannot build a communicator over it, and the same send/recv schedule
// runs as cudaMemcpyPeerAsync copies instead (transport "copy").
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <type_traits>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/nlgpu.h"

namespace {

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*asyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

const NcclApi* nccl_api(std::string& why) {
  static NcclApi api;
  static bool tried = false;
  static std::string err;
  if (!tried) {
    tried = true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.so = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.so) break;
    }
    if (!api.so) {
      err = std::string("NCCL not found (dlopen libnccl.so.2): ") + dlerror();
    } else {
      auto sym = [&](auto& fn, const char* s) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(api.so, s));
        if (!fn && err.empty()) err = std::string("NCCL symbol missing: ") + s;
      };
      sym(api.commInitAll, "ncclCommInitAll");
      sym(api.commDestroy, "ncclCommDestroy");
      sym(api.groupStart, "ncclGroupStart");
      sym(api.groupEnd, "ncclGroupEnd");
      sym(api.send, "ncclSend");
      sym(api.recv, "ncclRecv");
      sym(api.asyncError, "ncclCommGetAsyncError");
      sym(api.errorString, "ncclGetErrorString");
    }
  }
  why = err;
  return err.empty() ? &api : nullptr;
}

struct GError {
  nlg_status code;
  std::string msg;
};

#define G_CUDA(call)                                                                         \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) throw GError{NLG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

void check_plan(nlg_status st) {
  if (st != NLG_OK) throw GError{st, nlg_last_error()};
}

}  // namespace

struct nlg_group {
  int ndev = 0;
  bool use_nccl = false;
  const NcclApi* api = nullptr;
  std::vector<int> dev;
  std::vector<nlg_plan*> plan;
  std::vector<nlg_info> info;
  std::vector<int64_t> rb, re;          // owned rows per device
  int64_t n = 0, stride = 0;            // rows, nodes per row
  int comps = 1;
  std::vector<ncclComm_t> comm;
  std::vector<cudaStream_t> s, cs;       // compute / communication stream per device
  std::vector<cudaEvent_t> ev_u, ev_halo;
  std::vector<double*> u, out;           // device staging for the host entry point
};

namespace {

thread_local std::string g_err;

template <typename F>
nlg_status gguard(F&& f) {
  try {
    f();
    g_err.clear();
    return NLG_OK;
  } catch (const GError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NLG_ERUNTIME;
  }
}

void nccl_check(const nlg_group& G, ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw GError{NLG_ENCCL, std::string(what) + ": " + G.api->errorString(r)};
}

// Even split of n rows over ndev slabs (the first n % ndev get one more).
void slab(int64_t n, int ndev, int k, int64_t& rb, int64_t& re) {
  const int64_t base = n / ndev, extra = n % ndev;
  rb = k * base + std::min<int64_t>(k, extra);
  re = rb + base + (k < extra ? 1 : 0);
}

// u's halo exchange: device k receives rows [in_begin_k, rb_k) from k - 1 and
// [re_k, in_end_k) from k + 1, into the halo parts of its input buffer; every
// device sends the matching first / last owned rows. Enqueued on the
// communication streams after ev_u[k] (owned rows of u_k ready); records
// ev_halo[k].
void exchange(nlg_group& G, double* const* u) {
  const int nd = G.ndev;
  const size_t row = static_cast<size_t>(G.stride);
  for (int k = 0; k < nd; ++k) {
    G_CUDA(cudaSetDevice(G.dev[k]));
    G_CUDA(cudaStreamWaitEvent(G.cs[k], G.ev_u[k], 0));
  }
  // per component plane: [c][n_in_k]
  auto plane = [&](int k, int c) { return u[k] + static_cast<size_t>(c) * G.info[k].n_in; };
  if (G.use_nccl) {
    nccl_check(G, G.api->groupStart(), "ncclGroupStart");
    for (int k = 0; k < nd; ++k) {
      const int64_t lo = G.info[k].halo_lo, hi = G.info[k].halo_hi;
      const int64_t own = G.re[k] - G.rb[k];
      for (int c = 0; c < G.comps; ++c) {
        double* p = plane(k, c);
        if (k > 0 && lo > 0) nccl_check(G, G.api->recv(p, lo * row, ncclFloat64, k - 1, G.comm[k], G.cs[k]), "ncclRecv");
        if (k + 1 < nd && hi > 0)
          nccl_check(G, G.api->recv(p + (lo + own) * row, hi * row, ncclFloat64, k + 1, G.comm[k], G.cs[k]), "ncclRecv");
        if (k > 0) {   // the lower neighbour's halo_hi rows are my first owned rows
          const int64_t nh = G.info[k - 1].halo_hi;
          if (nh > 0) nccl_check(G, G.api->send(p + lo * row, nh * row, ncclFloat64, k - 1, G.comm[k], G.cs[k]), "ncclSend");
        }
        if (k + 1 < nd) {
          const int64_t nl = G.info[k + 1].halo_lo;
          if (nl > 0)
            nccl_check(G, G.api->send(p + (lo + own - nl) * row, nl * row, ncclFloat64, k + 1, G.comm[k], G.cs[k]),
                       "ncclSend");
        }
      }
    }
    nccl_check(G, G.api->groupEnd(), "ncclGroupEnd");
  } else {
    // copy transport: the receiver pulls from the neighbour's owned rows once
    // the neighbour's u is ready
    for (int k = 0; k < nd; ++k) {
      G_CUDA(cudaSetDevice(G.dev[k]));
      const int64_t lo = G.info[k].halo_lo, hi = G.info[k].halo_hi;
      const int64_t own = G.re[k] - G.rb[k];
      for (int c = 0; c < G.comps; ++c) {
        if (k > 0 && lo > 0) {
          G_CUDA(cudaStreamWaitEvent(G.cs[k], G.ev_u[k - 1], 0));
          const int64_t lo1 = G.info[k - 1].halo_lo, own1 = G.re[k - 1] - G.rb[k - 1];
          G_CUDA(cudaMemcpyPeerAsync(plane(k, c), G.dev[k], plane(k - 1, c) + (lo1 + own1 - lo) * row, G.dev[k - 1],
                                     sizeof(double) * lo * row, G.cs[k]));
        }
        if (k + 1 < nd && hi > 0) {
          G_CUDA(cudaStreamWaitEvent(G.cs[k], G.ev_u[k + 1], 0));
          const int64_t lo1 = G.info[k + 1].halo_lo;
          G_CUDA(cudaMemcpyPeerAsync(plane(k, c) + (lo + own) * row, G.dev[k], plane(k + 1, c) + lo1 * row, G.dev[k + 1],
                                     sizeof(double) * hi * row, G.cs[k]));
        }
      }
    }
  }
  for (int k = 0; k < nd; ++k) {
    G_CUDA(cudaSetDevice(G.dev[k]));
    G_CUDA(cudaEventRecord(G.ev_halo[k], G.cs[k]));
  }
}

void check_async(nlg_group& G) {
  if (!G.use_nccl) return;
  for (int k = 0; k < G.ndev; ++k) {
    ncclResult_t r = ncclSuccess;
    nccl_check(G, G.api->asyncError(G.comm[k], &r), "ncclCommGetAsyncError");
    nccl_check(G, r, "NCCL asynchronous error");
  }
}

// begin (halo-independent part) on s[k]; the exchange on cs[k]; end on s[k]
// after the halos landed
void apply_dev(nlg_group& G, double* const* u, double* const* out) {
  for (int k = 0; k < G.ndev; ++k) {
    G_CUDA(cudaSetDevice(G.dev[k]));
    G_CUDA(cudaEventRecord(G.ev_u[k], G.s[k]));
    check_plan(nlg_apply_fast_dev_begin(G.plan[k], u[k], out[k], G.s[k]));
  }
  exchange(G, u);
  for (int k = 0; k < G.ndev; ++k) {
    G_CUDA(cudaSetDevice(G.dev[k]));
    G_CUDA(cudaStreamWaitEvent(G.s[k], G.ev_halo[k], 0));
    check_plan(nlg_apply_fast_dev_end(G.plan[k], u[k], out[k], G.s[k]));
  }
}

void group_free(nlg_group* G) {
  if (!G) return;
  for (int k = 0; k < G->ndev; ++k) {
    if (k < static_cast<int>(G->dev.size())) cudaSetDevice(G->dev[k]);
    if (k < static_cast<int>(G->s.size()) && G->s[k]) cudaStreamSynchronize(G->s[k]);
    if (k < static_cast<int>(G->cs.size()) && G->cs[k]) cudaStreamSynchronize(G->cs[k]);
    if (k < static_cast<int>(G->plan.size())) nlg_plan_destroy(G->plan[k]);
    if (k < static_cast<int>(G->u.size())) cudaFree(G->u[k]);
    if (k < static_cast<int>(G->out.size())) cudaFree(G->out[k]);
    if (k < static_cast<int>(G->ev_u.size()) && G->ev_u[k]) cudaEventDestroy(G->ev_u[k]);
    if (k < static_cast<int>(G->ev_halo.size()) && G->ev_halo[k]) cudaEventDestroy(G->ev_halo[k]);
    if (k < static_cast<int>(G->s.size()) && G->s[k]) cudaStreamDestroy(G->s[k]);
    if (k < static_cast<int>(G->cs.size()) && G->cs[k]) cudaStreamDestroy(G->cs[k]);
  }
  if (G->use_nccl && G->api)
    for (ncclComm_t c : G->comm)
      if (c) G->api->commDestroy(c);
  delete G;
}

}  // namespace

extern "C" {

const char* nlg_group_last_error(void) { return g_err.c_str(); }

nlg_status nlg_group_create(const nlg_desc* desc, int ndev, const int* devices, nlg_group** out) {
  nlg_group* G = nullptr;
  const nlg_status st = gguard([&] {
    if (!desc || !devices || !out || ndev < 1) throw GError{NLG_EINVAL, "null argument or ndev < 1"};
    *out = nullptr;
    G = new nlg_group();
    G->ndev = ndev;
    G->dev.assign(devices, devices + ndev);
    G->n = desc->n;
    G->stride = 1;
    for (int j = 1; j < desc->dim; ++j) G->stride *= desc->n;
    G->comps = desc->family == NLG_PERIDYNAMIC ? desc->dim : 1;
    if (desc->row_end != 0) throw GError{NLG_EINVAL, "group descriptors cover the whole grid (row_end = 0)"};
    // halo rows and the slab split; every interior slab must be at least a halo deep
    double dmax = desc->delta0;
    const int64_t N = G->n * G->stride;
    if (desc->delta)
      for (int64_t i = 0; i < N; ++i) dmax = std::max(dmax, desc->delta[i]);
    int64_t halo = 0;
    check_plan(nlg_halo_rows(desc, dmax, &halo));
    if (ndev > 1) {
      for (int k = 0; k < ndev; ++k) {
        int64_t rb, re;
        slab(G->n, ndev, k, rb, re);
        if (re - rb < halo) throw GError{NLG_EINVAL, "slab thinner than the halo: use fewer devices"};
      }
    }
    std::vector<int> sorted(G->dev);
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    // NLG_GROUP_NCCL=1: a communicator even for one device (exercises the NCCL
    // set-up and error path on a single-GPU box)
    const char* force = std::getenv("NLG_GROUP_NCCL");
    G->use_nccl = distinct && (ndev > 1 || (force && std::atoi(force) == 1));
    if (G->use_nccl) {
      std::string why;
      G->api = nccl_api(why);
      if (!G->api) throw GError{NLG_ENCCL, why};
      G->comm.assign(ndev, nullptr);
      nccl_check(*G, G->api->commInitAll(G->comm.data(), ndev, G->dev.data()), "ncclCommInitAll");
    }
    G->plan.assign(ndev, nullptr);
    G->info.resize(ndev);
    G->rb.resize(ndev);
    G->re.resize(ndev);
    G->s.assign(ndev, nullptr);
    G->cs.assign(ndev, nullptr);
    G->ev_u.assign(ndev, nullptr);
    G->ev_halo.assign(ndev, nullptr);
    G->u.assign(ndev, nullptr);
    G->out.assign(ndev, nullptr);
    for (int k = 0; k < ndev; ++k) {
      int64_t rb, re;
      if (ndev > 1) slab(G->n, ndev, k, rb, re);
      else { rb = 0; re = G->n; }
      G->rb[k] = rb;
      G->re[k] = re;
      const int64_t ib = std::max<int64_t>(0, rb - halo), ie = std::min<int64_t>(G->n, re + halo);
      nlg_desc d = *desc;
      d.row_begin = rb;
      d.row_end = re;
      d.device = G->dev[k];
      if (ndev > 1 && d.reach <= 0.0) d.reach = dmax;   // the slab halo sized by the grid-wide horizon
      const int64_t off = ib * G->stride;
      if (desc->delta) d.delta = desc->delta + off;
      if (desc->coeff) d.coeff = desc->coeff + off;
      if (desc->kappa) d.kappa = desc->kappa + off;
      check_plan(nlg_plan_create(&d, &G->plan[k]));
      check_plan(nlg_plan_info(G->plan[k], &G->info[k]));
      if (G->info[k].halo_lo != rb - ib || G->info[k].halo_hi != ie - re)
        throw GError{NLG_ERUNTIME, "slab halo disagrees with the plan's"};
      G_CUDA(cudaSetDevice(G->dev[k]));
      G_CUDA(cudaStreamCreateWithFlags(&G->s[k], cudaStreamNonBlocking));
      G_CUDA(cudaStreamCreateWithFlags(&G->cs[k], cudaStreamNonBlocking));
      G_CUDA(cudaEventCreateWithFlags(&G->ev_u[k], cudaEventDisableTiming));
      G_CUDA(cudaEventCreateWithFlags(&G->ev_halo[k], cudaEventDisableTiming));
    }
    *out = G;
  });
  if (st != NLG_OK) group_free(G);
  return st;
}

void nlg_group_destroy(nlg_group* group) { group_free(group); }

nlg_status nlg_group_info(const nlg_group* G, int* ndev, int* nccl, int64_t* row_begin, int64_t* row_end,
                          int64_t* n_in) {
  return gguard([&] {
    if (!G || !ndev) throw GError{NLG_EINVAL, "null argument"};
    *ndev = G->ndev;
    if (nccl) *nccl = G->use_nccl ? 1 : 0;
    for (int k = 0; k < G->ndev; ++k) {
      if (row_begin) row_begin[k] = G->rb[k];
      if (row_end) row_end[k] = G->re[k];
      if (n_in) n_in[k] = G->info[k].n_in;
    }
  });
}

nlg_status nlg_group_apply_fast_dev(nlg_group* G, double* const* u_dev, double* const* out_dev) {
  return gguard([&] {
    if (!G || !u_dev || !out_dev) throw GError{NLG_EINVAL, "null argument"};
    apply_dev(*G, u_dev, out_dev);
    for (int k = 0; k < G->ndev; ++k) {
      G_CUDA(cudaSetDevice(G->dev[k]));
      G_CUDA(cudaStreamSynchronize(G->s[k]));
    }
    check_async(*G);
  });
}

nlg_status nlg_group_apply_fast(nlg_group* G, const double* u, double* out) {
  return gguard([&] {
    if (!G || !u || !out) throw GError{NLG_EINVAL, "null argument"};
    const size_t row = static_cast<size_t>(G->stride);
    const int64_t N = G->n * G->stride;
    for (int k = 0; k < G->ndev; ++k) {
      G_CUDA(cudaSetDevice(G->dev[k]));
      const nlg_info& I = G->info[k];
      if (!G->u[k]) G_CUDA(cudaMalloc(&G->u[k], sizeof(double) * G->comps * I.n_in));
      if (!G->out[k]) G_CUDA(cudaMalloc(&G->out[k], sizeof(double) * G->comps * I.n_out));
      // owned rows only: the halos come from the neighbours
      const int64_t own = G->re[k] - G->rb[k];
      for (int c = 0; c < G->comps; ++c)
        G_CUDA(cudaMemcpyAsync(G->u[k] + c * I.n_in + I.halo_lo * row, u + c * N + G->rb[k] * row,
                               sizeof(double) * own * row, cudaMemcpyHostToDevice, G->s[k]));
    }
    apply_dev(*G, G->u.data(), G->out.data());
    for (int k = 0; k < G->ndev; ++k) {
      G_CUDA(cudaSetDevice(G->dev[k]));
      const nlg_info& I = G->info[k];
      for (int c = 0; c < G->comps; ++c)
        G_CUDA(cudaMemcpyAsync(out + c * N + G->rb[k] * row, G->out[k] + c * I.n_out, sizeof(double) * I.n_out,
                               cudaMemcpyDeviceToHost, G->s[k]));
    }
    for (int k = 0; k < G->ndev; ++k) {
      G_CUDA(cudaSetDevice(G->dev[k]));
      G_CUDA(cudaStreamSynchronize(G->s[k]));
    }
    check_async(*G);
  });
}

}  // extern "C"
