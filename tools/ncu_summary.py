"""Summarise ncu outputs into profiles/ (run here, after gpurun brings them back).

  python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <workload> <tag>

Writes profiles/<tag>_launches.json (per-kernel launch counts, total and mean
device time, share), profiles/<tag>_ncu_full.json (key metrics of the captured
kernels) and updates profiles/ncu_traffic.json[workload] with the DRAM bytes
per launch of the dominant captured kernel (bench.py reads it for
roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("nlg::<unnamed>::", "")
        v = float(r[vi].replace(",", ""))
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    return {k: {"launches": cnt[k], "total_ns": tot[k], "mean_ns": tot[k] / cnt[k], "share": tot[k] / total}
            for k in sorted(tot, key=lambda x: -tot[x])}


KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__inst_executed.sum"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    units = rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = r[i] + ("" if not units[i] else f" {units[i]}")
        res.append(d)
    return res


def to_bytes(s):
    v, _, unit = s.partition(" ")
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


# kernel name -> bench.py stage (nlg stage names, _capi.STAGES)
def stage_of(name):
    import re
    n = name.replace("void ", "").replace("nlg::<unnamed>::", "").replace("<unnamed>::", "")
    rules = [(r"f3_ties", "box_ties"), (r"f3_rows<\d+, 0", "box_pa_rows_fwd"), (r"f3_rows<\d+, 1", "box_pe_rows_inv"),
             (r"f3_cols(_tma)?<\d+, 0", "box_pb_cols_fwd"), (r"f3_cols(_tma)?<\d+, 1", "box_pd_cols_inv"),
             (r"f3_zstencil", "box_pc_zstencil"), (r"es_tail_walk<\d+, 1", "es_main"),
             (r"es_tail_walk<\d+, 0", "es_aggregate"), (r"es_carry", "es_carry"), (r"cols_fwd", "es_fft_p1_cols_fwd"),
             (r"fs_rows", "es_fft_p2_rows"), (r"cols_inv", "es_fft_p3_cols_inv"), (r"es_fft_combine", "es_combine"),
             (r"stencil", "stencil"), (r"direct", "direct"), (r"scan_lookback|moment_scan", "span_scan"),
             (r"span_eval|moment_eval", "span_eval")]
    for pat, st in rules:
        if re.search(pat, n):
            return st
    return n


def main():
    if sys.argv[1] == "--r02":
        return main_r02(sys.argv[2:])
    lpath, fpath, workload, tag = sys.argv[1:5]
    os.makedirs(PROF, exist_ok=True)
    L = launches(lpath)
    json.dump(L, open(os.path.join(PROF, f"{tag}_launches.json"), "w"), indent=1)
    F = full(fpath)
    json.dump(F, open(os.path.join(PROF, f"{tag}_ncu_full.json"), "w"), indent=1)
    tp = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    if F:
        dom = max(F, key=lambda d: float(d["gpu__time_duration.sum"].split()[0].replace(",", "")))
        traffic[workload] = {"kernel": dom["Kernel Name"],
                             "dram_bytes_per_launch": to_bytes(dom["dram__bytes_read.sum"]) +
                             to_bytes(dom["dram__bytes_write.sum"]),
                             "source": f"profiles/{tag}_ncu_full.json"}
        json.dump(traffic, open(tp, "w"), indent=1)
    print(json.dumps({"launches": L, "traffic": traffic.get(workload)}, indent=1))


def main_r02(argv):
    """ncu_summary.py --r02 <launches.csv|-> <full.ncu-rep> <workload key> <tag>: every
    captured kernel keyed by its bench stage; ncu_traffic.json[workload][stage] =
    dram read+write bytes per launch."""
    lpath, fpath, workload, tag = argv[:4]
    os.makedirs(PROF, exist_ok=True)
    res = {"workload": workload}
    if lpath != "-":
        L = launches(lpath)
        res["launches"] = L
        json.dump(L, open(os.path.join(PROF, f"{tag}_launches.json"), "w"), indent=1)
    F = full(fpath)
    for d in F:
        d["stage"] = stage_of(d["Kernel Name"])
    json.dump(F, open(os.path.join(PROF, f"{tag}_ncu_full.json"), "w"), indent=1)
    tp = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    ent = traffic.get(workload) if isinstance(traffic.get(workload), dict) and "kernel" not in traffic.get(workload, {}) else {}
    for d in F:
        if "dram__bytes_read.sum" in d:
            ent[d["stage"]] = {"bytes": to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"]),
                               "kernel": d["Kernel Name"], "source": f"profiles/{tag}_ncu_full.json"}
    traffic[workload] = ent
    json.dump(traffic, open(tp, "w"), indent=1)
    print(json.dumps({k: v["bytes"] for k, v in ent.items()}, indent=1))


if __name__ == "__main__":
    main()
