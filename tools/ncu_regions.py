"""Per-region summary of an ncu report's SASS source page + key raw metrics.

usage: python tools/ncu_regions.py <report.ncu-rep> [bucket=100]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
bucket = int(sys.argv[2]) if len(sys.argv) > 2 else 100
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
h, rows = r[1], r[2:]
isrc, ie, iss = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
iw, iwi = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
tot = sum(int(x[ie]) for x in rows) or 1
st = sum(int(x[iss]) for x in rows) or 1
tw = sum(int(x[iw]) for x in rows) or 1
print("instructions", tot, "smem wavefronts", tw)
for b in range(0, len(rows), bucket):
    seg = rows[b:b + bucket]
    a = sum(int(x[ie]) for x in seg)
    s = sum(int(x[iss]) for x in seg)
    nd = sum(int(x[ie]) for x in seg if "DFMA" in x[isrc] or "DADD" in x[isrc] or "DMUL" in x[isrc])
    w = sum(int(x[iw]) for x in seg)
    wi = sum(int(x[iwi]) for x in seg)
    if a / tot > 0.005 or s / st > 0.01:
        print(f"{b:5d} inst {a / tot:6.1%} stall {s / st:6.1%} fp64 {nd / tot:6.1%} wf {w / tw:6.1%} "
              f"(ideal {wi / tw:6.1%})  {seg[0][isrc].strip()[:44]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, v = rr[0], rr[-1]
stalls = []
for i, name in enumerate(h):
    if "pcsamp_warps_issue_stalled" in name and not name.endswith("not_issued"):
        try:
            stalls.append((float(v[i].replace(",", "")), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
ts = sum(x[0] for x in stalls) or 1
print("stalls:", ", ".join(f"{n} {c / ts:.0%}" for c, n in sorted(stalls, reverse=True)[:8]))
keys = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem"]
for k in keys:
    if k in h:
        print(k, v[h.index(k)])
