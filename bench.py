"""bench.py — fp64 nonlocal-apply throughput (BASELINE.json metric) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg1] [--impl ours|reference]

One step = one fast apply of the whole workload (default BASELINE configs[1]:
1-D N=2^22, variable delta, kappa-weighted fractional kernel, s=0.4) with the
inputs resident in HBM. N>1 runs one process per GPU (torchrun), slabs along
axis 0 with NCCL halo exchange every step (strong scaling: the total grid is
fixed). L2 (126 MB) is flushed with a 256 MB write between timed steps; each
step is timed on the device with CUDA events on the plan's stream; the job
time is the max over ranks.

Extra keys: roofline (whole fast apply and the
dominant kernel, live CUDA-event stage times), cpu_baseline (the compiled
reference on the host cores, bounded sample), e2e (public host API incl.
H2D/D2H), clocks (NVML during the timed region), gpu_launches.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 nonlocal-apply grid points/s (1/2/4/8 B200); % HBM roofline"
UNIT = "grid points/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _dfma_peak():
    try:
        with open(os.path.join(ROOT, "profiles", "dfma_peak.json")) as f:
            return float(json.load(f)["dfma_tflops"])
    except Exception:
        return None


def _traffic(workload):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload)
    except Exception:
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


def _workload(name):
    from paper_1905_08375_b200 import configs
    return configs.WORKLOADS[name]()


def _cpu_reference(w, seconds_budget: float, nthreads: int, seed: int = 11):
    """The compiled reference (oracle/_ref) on a bounded random sample of the
    workload's output nodes; falls back to the restated oracle ("port")."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    rng = np.random.default_rng(seed)
    if O.ref_available() and w.kernel == "fractional":
        kind = "reference"
        delta = w.delta if w.delta is not None else np.full(w.N, w.delta0)
        cx = w.coeff if w.coeff is not None else np.full(w.N, w.coeff0)

        def run(tg):
            return O.ref_full_dense_general_at(w.dim, w.n, delta, cx, w.kappa, w.alpha, w.u, tg,
                                               nthreads=nthreads)
    else:
        kind = "port"
        nthreads = 1

        def run(tg):
            return O.apply(w.dim, w.n, w.u, targets=tg, **w.oracle_kwargs())
    # calibrate the sample so one run takes ~seconds_budget
    cnt, el = 16, 0.0
    while True:
        tg = rng.integers(0, w.N, cnt)
        t0 = time.perf_counter()
        run(tg)
        el = time.perf_counter() - t0
        if el > 0.25 * seconds_budget or cnt >= w.N:
            break
        cnt = min(w.N, cnt * 4)
    cnt = int(min(w.N, max(cnt, cnt * seconds_budget / max(el, 1e-6))))
    tg = rng.integers(0, w.N, cnt)
    t0 = time.perf_counter()
    run(tg)
    el = time.perf_counter() - t0
    return {"value": cnt / el, "unit": UNIT, "cores": nthreads, "kind": kind,
            "sample": f"{cnt} random output nodes of {w.name} (of {w.N}), {el:.2f} s, "
                      f"apply_full_dense per-node loop + eval_omega"
                      if kind == "reference" else f"{cnt} random nodes, restated oracle, {el:.2f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = _workload(args.workload)
    nthreads = os.cpu_count() or 1
    vals = []
    base = None
    for k in range(args.warmup + args.steps):
        r = _cpu_reference(w, args.ref_seconds, nthreads, seed=100 + k)
        if k >= args.warmup:
            vals.append(r["value"])
            base = r
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
        "config": {"workload": w.name, "dim": w.dim, "n": w.n, "N": w.N, "alpha": w.alpha,
                   "exterior": "collar" if w.exterior else "clip"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": base["cores"], "kind": base["kind"],
                         "sample": base["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1905_08375_b200 import nonloc as NL
    from paper_1905_08375_b200.slabs import Slab

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    w = _workload(args.workload)
    stride = w.n ** (w.dim - 1)
    dmax = float(w.delta.max()) if w.delta is not None else w.delta0
    halo = NL.halo_rows(dim=w.dim, n=w.n, family=4 if w.kernel == "fractional" else 5, delta_max=dmax)
    sl = Slab(w.n, stride, halo if world > 1 else 0, rank, world)
    kw = w.op_kwargs()
    for key in ("delta", "coeff", "kappa"):
        kw[key] = sl.input_slice(kw[key])
    t_plan = time.perf_counter()
    op = NL.NonlocalOperator(w.dim, w.n, row_begin=sl.row_begin, row_end=sl.row_end,
                             reach=dmax if world > 1 else 0.0, device=local, **kw)
    t_plan = time.perf_counter() - t_plan
    plan = op.plan
    comps = plan.components
    u_full = w.u
    u_in_host = sl.input_slice(u_full) if comps == 1 else np.concatenate(
        [sl.input_slice(u_full[c * w.N:(c + 1) * w.N]) for c in range(comps)])
    u_in = torch.from_numpy(u_in_host).to(dev)
    out = torch.empty(comps * plan.n_out, dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        if world > 1:
            sl.exchange(u_in)
        plan.apply_fast_dev(u_in.data_ptr(), out.data_ptr(), stream.cuda_stream)

    # warm-up (W >= 3 enforced by the driver's rules)
    for _ in range(max(args.warmup, 1)):
        with torch.cuda.stream(stream):
            step()
    torch.cuda.synchronize()

    # timed region: per-step CUDA events on the plan stream, L2 flushed between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = plan.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local).start()
    # everything is enqueued on one stream without host syncs, so the host runs
    # ahead (the flush covers the launch latency) and no host gap is timed
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
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = w.N / (ms_step * 1e-3)   # output grid points (all components) per second

    # dominant kernel: live CUDA-event stage times over a few extra applies
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
    A = NL.A
    import ctypes as C
    up = C.cast(u_host.data_ptr(), A._dp)
    op_ = C.cast(out_host.data_ptr(), A._dp)
    A.check(A.lib().nlg_apply_fast(plan._h, up, op_))
    e2e_s = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        A.check(A.lib().nlg_apply_fast(plan._h, up, op_))
        e2e_s.append(time.perf_counter() - t0)
    e2e_step = sum(e2e_s) / len(e2e_s)
    te = torch.tensor([e2e_step], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = w.N / float(te.item())

    if rank == 0:
        peak, peak_kind = _peaks()
        bpp = w.bytes_per_point()
        achieved = bpp * (w.N / world) / (ms_step * 1e-3) / 1e9   # per GPU, whole fast apply
        stage_avg = {k: v[0] / max(v[1], 1) for k, v in stages.items()}
        stage_share = {k: v[0] / max(sum(x[0] for x in stages.values()), 1e-12) for k, v in stages.items()}
        dom = max(stages.items(), key=lambda kv: kv[1][0])[0] if stages else None
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": _traffic(w.name),
                "peak_source": peak_kind,
                "scope": "whole fast apply (all kernels of one step), algorithmic "
                         f"{bpp} B/pt x {w.N // world} pts per GPU",
                "dominant_kernel": dom, "stage_ms_per_launch": stage_avg, "stage_share": stage_share}
        dfma = _dfma_peak()
        if dfma:
            roof["fp64_peak_tflops_measured"] = dfma
            info = plan.info
            if int(info.fast_method) == 2 and int(info.fft_len) > 0:
                # the 1-D path's algorithmic fp64 work: the four-step
                # convolution, 2 x 5 L log2 L, and the tail walks, 4 DFMA (aggregate 1 +
                # main 3) per term, field, node and direction
                import math
                L = int(info.fft_len)
                nf = 2 if w.kappa is not None else 1
                flops = 2 * 5 * L * math.log2(L) + 2 * 4 * int(info.exp_terms) * nf * 2 * plan.n_in
                tf = flops / (ms_step * 1e-3) / 1e12
                roof["fp64"] = {"achieved_tflops": tf, "peak_tflops": dfma, "frac": tf / dfma,
                                "flop_per_apply": flops,
                                "scope": "FFT 10 L log2 L + tail walks 8 M nf N (2 directions)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "config": {"workload": w.name, "dim": w.dim, "n": w.n, "N": w.N, "alpha": w.alpha,
                       "s": w.s, "exterior": "collar" if w.exterior else "clip", "seeds": w.seeds,
                       "parallelism": f"slab{world}", "l2": "flushed (256 MB write) between timed steps",
                       "fast_method": int(plan.info.fast_method), "exp_terms": int(plan.info.exp_terms),
                       "far_rel_err": float(plan.info.far_rel_err), "plan_seconds": t_plan},
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(u_host.numel() * 8),
                    "d2h_bytes_per_step": int(out_host.numel() * 8)},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = _cpu_reference(w, args.ref_seconds, os.cpu_count() or 1)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-seconds", type=float, default=1.5,
                    help="CPU seconds (wall) per reference sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
