"""bench.py — fp64 nonlocal-apply throughput (BASELINE.json metric) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--extra cfg4b,cfg2,cfg3,cfg1,trunc1d,trunc2d]
                  [--impl ours|reference]

One step = one fast apply of the whole workload with the inputs resident in
HBM. The headline workload is the largest BASELINE configuration that fits one
B200: configs[4] at 768^3 with the constant horizon delta = 6h (cfg4-A: 3-D,
kappa-weighted fractional kernel, s = 0.25). cfg4-B (variable horizon), cfg2
and cfg3 (2-D, 4096^2), cfg1 (1-D, N = 2^22) and the reference's own fast route
(TruncatedOperator, K = 0: trunc1d at 2^22, trunc2d at 1024^2) are measured in
the same run and carried under "extra".

N > 1: one process per GPU. Without WORLD_SIZE in the environment bench.py
re-launches itself under torch.distributed.run with N ranks (and fails loudly
when fewer than N GPUs are visible). Each rank owns a slab of axis-0 rows
(SURVEY §8(e)); u's halo rows move by NCCL point-to-point every step,
overlapped with the part of the apply that does not read them. The total grid
is fixed: strong scaling.

Timing: L2 (126 MB) flushed with a 256 MB write before every timed step; each
step bracketed by CUDA events on the plan's stream; job time = max over ranks.

Extra keys: roofline (dominant kernel from per-kernel CUDA-event
times of a serialized profiling pass; the whole apply beside it), cpu_baseline
(the compiled reference on the host cores over a FIXED target set, 1 core and
all cores), e2e (the public host entry nlg_apply_fast, pinned host buffers,
H2D + D2H inside the timed region), clocks (NVML during the timed region),
gpu_launches.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 nonlocal-apply grid points/s (1/2/4/8 B200); % HBM roofline"
UNIT = "grid points/s"
TARGET_SEED = 20261020          # the fixed CPU-baseline target set

# Fixed CPU-baseline samples (output nodes): one-core leg, all-cores leg.
# Sized for ~1-3 s of wall time each on the GPU box's host (16 threads);
# large enough that thread start-up and scheduling noise stay small.
CPU_SAMPLE = {"cfg0": (4096, 4096), "cfg1": (128, 2048), "cfg2": (16384, 262144), "cfg3": (16384, 131072),
              "cfg4": (4096, 65536), "cfg4b": (2048, 32768)}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _dfma_peak():
    try:
        with open(os.path.join(ROOT, "profiles", "dfma_peak.json")) as f:
            return float(json.load(f)["dfma_tflops"])
    except Exception:
        return None


def _traffic(keys, kernel):
    """ncu dram bytes (read + write) per launch of the stage `kernel` for the
    workload (any of `keys`), from a committed `ncu --set full` capture
    (profiles/ncu_traffic.json, written by tools/ncu_summary.py --r02), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
    except Exception:
        return None
    for k in keys:
        e = t.get(k)
        if isinstance(e, dict) and isinstance(e.get(kernel), dict):
            return e[kernel].get("bytes")
    return None


class ClockSampler:
    """NVML clocks + throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self._N = N
            self._h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM)
        except Exception:
            self._N = None
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        N = self._N
        names = {
            getattr(N, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(N, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(N, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(N, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(N, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self._h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.002)   # several samples even in a ~10 ms timed region

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def _workload(name, rows=None):
    from paper_1905_08375_b200 import configs
    return configs.WORKLOADS[name]()


# ---------------------------------------------------------------------------
# CPU reference (test infrastructure: the only place bench.py runs oracle/)
# ---------------------------------------------------------------------------

def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    return O


def _fixed_targets(N, count):
    """The fixed CPU-baseline target set: `count` distinct output nodes drawn
    with TARGET_SEED, in draw order (a prefix is itself a uniform sample)."""
    rng = np.random.default_rng(TARGET_SEED)
    return rng.choice(N, size=min(count, N), replace=False).astype(np.int64)


class DirectReference:
    """apply_full_dense per-node loop + eval_omega (operators.cpp:236-260,
    kernel.cpp:275-287) with the coefficient_fn emulation of the fractional /
    kappa / variable-delta kernel, compiled from the unmodified reference
    sources (oracle/_ref), over a FIXED target set: a one-core leg and an
    all-cores leg. The reference requires n = 2^L (geometry.cpp:14-16); for
    cfg4's 768^3 it runs on the 512^3 twin: its per-point cost depends only on
    delta/h (the window holds (2 ceil(delta/h) + 3)^3 candidates), so the twin
    keeps delta/h, s and the kappa weighting, with the 768^3 fields resampled at
    the nearest node and filled only where the sampled targets read them.
    Peridynamics (cfg3) has no reference: the restated oracle ("port")."""

    def __init__(self, w, key, nthreads):
        self.O = _oracle()
        self.w = w
        self.nthreads = nthreads
        c1, cn = CPU_SAMPLE.get(key, (1024, 8192))
        self.port = w.kernel == "peridynamic" or not self.O.ref_available()
        if self.port:
            self.t1 = _fixed_targets(w.N, c1)
            self.desc = f"{w.name}"
            return
        n = 1 << int(math.floor(math.log2(w.n)))
        if n == w.n:
            self.n = w.n
            self.delta = w.delta if w.delta is not None else np.full(w.N, w.delta0)
            self.cx = w.coeff if w.coeff is not None else np.full(w.N, w.coeff0)
            self.u, self.kappa = w.u, w.kappa
            self.tn = _fixed_targets(w.N, cn)
            self.desc = w.name
        else:
            self._twin(n, cn)
        self.t1 = self.tn[:c1]

    def _twin(self, n, cn):
        from paper_1905_08375_b200.nonloc import fractional_cdelta
        w = self.w
        d = w.dim
        N = n ** d
        idx = np.minimum(((np.arange(n) + 0.5) / n * w.n).astype(np.int64), w.n - 1)
        stride = [w.n ** (d - 1 - j) for j in range(d)]

        def src_index(flat):
            k = np.unravel_index(flat, (n,) * d)
            return sum(idx[k[j]] * stride[j] for j in range(d))

        self.n = n
        self.u = np.zeros(N)
        self.kappa = np.zeros(N) if w.kappa is not None else None
        self.delta = np.zeros(N)
        self.cx = np.zeros(N)
        self.tn = _fixed_targets(N, cn)
        D = int(math.ceil((w.delta.max() if w.delta is not None else w.delta0) * w.n)) + 2
        offs = np.arange(-D, D + 1)
        cube = np.stack(np.meshgrid(*([offs] * d), indexing="ij"), -1).reshape(-1, d)
        k = np.stack(np.unravel_index(self.tn, (n,) * d), axis=1)
        for j in range(0, len(k), 256):          # every node a sampled target's window reads
            nb = (k[j:j + 256, None, :] + cube[None, :, :]).reshape(-1, d)
            nb = nb[np.all((nb >= 0) & (nb < n), axis=1)]
            flat = np.ravel_multi_index(nb.T, (n,) * d)
            s = src_index(flat)
            self.u[flat] = w.u[s]
            if self.kappa is not None:
                self.kappa[flat] = w.kappa[s]
        s = src_index(self.tn)
        dd = (w.delta[s] if w.delta is not None else np.full(len(s), w.delta0)) * (w.n / n)
        self.delta[self.tn] = dd
        self.cx[self.tn] = fractional_cdelta(d, w.s, dd)
        self.desc = f"{w.name} on its {n}^{d} twin (delta/h, s, kappa weighting kept)"

    def _run(self, tg, nth):
        t0 = time.perf_counter()
        if self.port:
            self.O.apply(self.w.dim, self.w.n, self.w.u, targets=tg, **self.w.oracle_kwargs())
        else:
            self.O.ref_full_dense_general_at(self.w.dim, self.n, self.delta, self.cx, self.kappa, self.w.alpha,
                                             self.u, tg, nthreads=nth)
        return time.perf_counter() - t0

    def measure(self):
        if self.port:
            e1 = self._run(self.t1, 1)
            v = len(self.t1) / e1
            return {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "value_1core": v,
                    "sample": f"{len(self.t1)} fixed output nodes (seed {TARGET_SEED}) of {self.desc}, "
                              f"restated oracle (oracle/nonloc_oracle.c), 1 core, {e1:.2f} s"}
        self._run(self.t1[:4], 1)                # page in
        e1 = self._run(self.t1, 1)
        en = self._run(self.tn, self.nthreads)
        return {"value": len(self.tn) / en, "unit": UNIT, "cores": self.nthreads, "kind": "reference",
                "value_1core": len(self.t1) / e1,
                "sample": f"fixed output nodes (seed {TARGET_SEED}) of {self.desc}: {len(self.tn)} on "
                          f"{self.nthreads} threads ({en:.2f} s), the first {len(self.t1)} of them on 1 core "
                          f"({e1:.2f} s); apply_full_dense per-node loop + eval_omega, compiled unmodified "
                          f"reference (oracle/_ref)"}


def _cpu_reference_trunc(w, reps):
    """TruncatedOperator::apply (Steps 2+3, bench.cpp:47-49) of the compiled
    reference on the whole grid; Step 1 (the constructor) reported apart.
    The reference is single-threaded."""
    O = _oracle()
    _, cnt, tm = O.ref_truncated_fast(w.dim, w.n, w.K, w.horizon_kind, w.delta0, w.u, coeff=w.coeff0, reps=reps)
    v = w.N / tm[1]
    return {"value": v, "unit": UNIT, "cores": 1, "kind": "reference", "value_1core": v,
            "step1_seconds": float(tm[0]), "apply_seconds": float(tm[1]),
            "sample": f"whole grid of {w.name}, mean of {reps} TruncatedOperator::apply calls "
                      f"(Steps 2+3), Step 1 {tm[0]:.1f} s excluded; compiled unmodified reference"}


def cpu_reference(w, key, reps=1, steps=1, warmup=0):
    """Returns one measurement per step (after `warmup` untimed ones)."""
    if w.kernel == "truncated":
        return [_cpu_reference_trunc(w, reps) for _ in range(steps)]
    ref = DirectReference(w, key, os.cpu_count() or 1)
    for _ in range(warmup):
        ref.measure()
    return [ref.measure() for _ in range(steps)]


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = _workload(args.workload)
    rs = cpu_reference(w, args.workload, steps=args.steps, warmup=args.warmup)
    value = statistics.mean(r["value"] for r in rs)
    base = rs[-1]
    cpu = {k: base[k] for k in ("kind", "cores", "sample") if k in base}
    cpu.update({"value": value, "unit": UNIT,
                "value_1core": statistics.mean(r["value_1core"] for r in rs)})
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
        "config": _config(w, 1), "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def _config(w, world):
    c = {"workload": w.name, "dim": w.dim, "n": w.n, "N": w.N, "kernel": w.kernel, "seeds": w.seeds,
         "parallelism": f"slab{world}", "l2": "flushed (256 MB write) before every timed step"}
    if w.kernel == "truncated":
        c.update({"K": w.K, "horizon": "gaussian_bump" if w.horizon_kind else "constant", "delta0": w.delta0,
                  "rule": "leaf", "form": "mass"})
    else:
        c.update({"alpha": w.alpha, "s": w.s, "exterior": "collar" if w.exterior else "clip",
                  "horizon": "variable" if w.delta is not None else f"constant {w.delta0 * w.n:g}h"})
    return c


def _make_plan(w, sl, world, device):
    from paper_1905_08375_b200 import nonloc as NL
    if w.kernel == "truncated":
        spec = NL.KernelSpec(w.dim, NL.RadialProfile.truncated_polynomial(w.K),
                             NL.HorizonField(NL.HorizonKind(w.horizon_kind), w.delta0))
        if world > 1:
            raise SystemExit("truncated workloads run on one GPU")
        return NL.TruncatedOperator(spec, NL.Grid.make(w.dim, w.n), device=device)._plan
    kw = w.op_kwargs()
    for key in ("delta", "coeff", "kappa"):
        kw[key] = sl.input_slice(kw[key])
    dmax = float(w.delta.max()) if w.delta is not None else w.delta0
    return NL.NonlocalOperator(w.dim, w.n, row_begin=sl.row_begin, row_end=sl.row_end,
                               reach=dmax if world > 1 else 0.0, device=device, **kw).plan


def measure(name, args, world, rank, local, dev, full=True):
    """Device-timed fast apply of one workload: value, e2e, per-kernel times."""
    import torch
    import torch.distributed as dist
    from paper_1905_08375_b200 import nonloc as NL
    from paper_1905_08375_b200.slabs import Slab, slab_apply

    w = _workload(name)
    stride = w.n ** (w.dim - 1)
    dmax = float(w.delta.max()) if w.delta is not None else w.delta0
    if w.kernel == "truncated":
        halo = 0
    else:
        halo = NL.halo_rows(dim=w.dim, n=w.n, family=4 if w.kernel == "fractional" else 5, delta_max=dmax)
    sl = Slab(w.n, stride, halo if world > 1 else 0, rank, world)
    t_plan = time.perf_counter()
    plan = _make_plan(w, sl, world, local)
    t_plan = time.perf_counter() - t_plan
    comps = plan.components
    u_in_host = sl.input_slice(w.u) if comps == 1 else np.concatenate(
        [sl.input_slice(w.u[c * w.N:(c + 1) * w.N]) for c in range(comps)])
    u_in = torch.from_numpy(u_in_host).to(dev)
    out = torch.empty(comps * plan.n_out, dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        if world > 1:
            # halo-independent part first, u's halos in flight meanwhile
            slab_apply(sl, plan, u_in, out, stream.cuda_stream)
        else:
            plan.apply_fast_dev(u_in.data_ptr(), out.data_ptr(), stream.cuda_stream)

    for _ in range(max(args.warmup, 1)):
        with torch.cuda.stream(stream):
            step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = plan.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local).start()
    # enqueued on one stream without host syncs: the host runs ahead (the
    # flush covers the launch latency), no host gap is timed
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            flush.fill_(float(k))
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    launches = plan.launch_count() - launches0
    ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    value = w.N / (ms_step * 1e-3)   # output grid points (all components) per second, all ranks

    # per-kernel times: a serialized profiling pass (side streams folded in)
    stages = {}
    if full:
        plan.set_profiling(True)
        plan.stage_times()
        with torch.cuda.stream(stream):
            for _ in range(3):
                flush.fill_(0.0)
                plan.apply_fast_dev(u_in.data_ptr(), out.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        stages = plan.stage_times()
        plan.set_profiling(False)

    # e2e through the public host API (H2D of u, D2H of out inside the timed region)
    u_host = torch.from_numpy(u_in_host).pin_memory()
    out_host = torch.empty(comps * plan.n_out, dtype=torch.float64).pin_memory()
    plan.apply_fast_host_ptr(u_host.data_ptr(), out_host.data_ptr())
    e2e_s = []
    for _ in range(args.steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        plan.apply_fast_host_ptr(u_host.data_ptr(), out_host.data_ptr())
        e2e_s.append(time.perf_counter() - t0)
    te = torch.tensor([sum(e2e_s) / len(e2e_s)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": w.N / float(te.item()), "unit": UNIT,
           "h2d_bytes_per_step": int(u_host.numel() * 8) * world,
           "d2h_bytes_per_step": int(out_host.numel() * 8) * world,
           "path": "nlg_apply_fast (host pointers; plane-chunked H2D / apply / D2H pipeline where the "
                   "method supports it)"}

    res = {"key": name, "w": w, "plan": plan, "value": value, "ms_per_step": ms_step, "e2e": e2e, "stages": stages,
           "launches": launches, "clocks": clk, "plan_seconds": t_plan, "n_out": plan.n_out}
    del u_in, out, flush
    return res


def _roofline(res, world):
    w, plan = res["w"], res["plan"]
    peak, peak_kind = _peaks()
    bpp = w.bytes_per_point()
    units = w.N // world
    apply_gbs = bpp * units / (res["ms_per_step"] * 1e-3) / 1e9
    st = res["stages"]
    per_launch = {k: v[0] / max(v[1], 1) for k, v in st.items()}
    tot = sum(v[0] for v in st.values())
    share = {k: v[0] / tot for k, v in st.items()} if tot > 0 else {}
    dom = max(st.items(), key=lambda kv: kv[1][0])[0] if st else None
    roof = {"bound": "hbm", "peak": peak, "unit": "GB/s", "peak_source": peak_kind}
    if dom:
        # contract: algorithmic bytes of one launch (B/pt x points) / that
        # kernel's average launch duration (CUDA events, serialized pass)
        dom_ms = per_launch[dom]
        ach = bpp * units / (dom_ms * 1e-3) / 1e9
        roof.update({"achieved": ach, "frac": ach / peak, "traffic": _traffic((res["key"], w.name), dom),
                     "dominant_kernel": dom, "dominant_ms_per_launch": dom_ms,
                     "dominant_share": share[dom],
                     "scope": f"dominant kernel: algorithmic {bpp} B/pt x {units} pts per launch / its mean "
                              f"launch time; traffic = ncu dram read+write per launch of that kernel"})
    else:
        roof.update({"achieved": apply_gbs, "frac": apply_gbs / peak, "traffic": None})
    roof["apply"] = {"achieved": apply_gbs, "frac": apply_gbs / peak,
                     "scope": f"whole fast apply (all kernels of one step): {bpp} B/pt x {units} pts"}
    roof["kernel_ms_per_launch"] = per_launch
    roof["kernel_share"] = share
    dfma = _dfma_peak()
    if dfma:
        roof["fp64_peak_tflops_measured"] = dfma
        info = plan.info
        if int(info.fast_method) == 2 and int(info.fft_len) > 0:
            L = int(info.fft_len)
            nf = 2 if w.kappa is not None else 1
            flops = 2 * 5 * L * math.log2(L) + 2 * 4 * int(info.exp_terms) * nf * 2 * plan.n_in
            tf = flops / (res["ms_per_step"] * 1e-3) / 1e12
            roof["fp64"] = {"achieved_tflops": tf, "peak_tflops": dfma, "frac": tf / dfma,
                            "flop_per_apply": flops,
                            "scope": "FFT 10 L log2 L + tail walks 8 M nf N (2 directions)"}
    return roof


def _summary(res, world):
    w = res["w"]
    roof = _roofline(res, world)
    return {"workload": w.name, "value": res["value"], "unit": UNIT, "ms_per_step": res["ms_per_step"],
            "e2e": res["e2e"], "roofline_frac": roof["frac"], "apply_hbm_frac": roof["apply"]["frac"],
            "dominant_kernel": roof.get("dominant_kernel"), "kernel_ms_per_launch": roof["kernel_ms_per_launch"],
            "gpu_launches": res["launches"], "config": _config(w, world)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    main = measure(args.workload, args, world, rank, local, dev)
    roof = _roofline(main, world)
    w = main["w"]
    cfg = _config(w, world)
    cfg.update({"fast_method": int(main["plan"].info.fast_method), "plan_seconds": main["plan_seconds"]})
    if int(main["plan"].info.fft_len):
        cfg["fft_len"] = int(main["plan"].info.fft_len)
    line = {
        "metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": main["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
        "config": cfg, "roofline": roof, "e2e": main["e2e"], "gpu_launches": int(main["launches"]),
        "clocks": main["clocks"],
    }
    plan_main = main.pop("plan")
    del plan_main
    extras = {}
    for name in [x for x in args.extra.split(",") if x]:
        if world > 1 and name in ("trunc1d", "trunc2d"):
            continue
        r = measure(name, args, world, rank, local, dev)
        extras[name] = _summary(r, world)
        del r
        torch.cuda.empty_cache()
    if extras:
        line["extra"] = extras
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_reference(w, args.workload)[0]
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _self_launch(args):
    """--gpus N without a torchrun environment: re-exec under
    torch.distributed.run with N ranks (one per GPU)."""
    import socket
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:
        have = 0
    if have < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} requested but {have} GPU(s) visible")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--extra", default="cfg4b,cfg2,cfg3,cfg1,trunc1d,trunc2d",
                    help="comma-separated workloads measured after the headline ('' for none)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _self_launch(args)
    if args.gpus > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
