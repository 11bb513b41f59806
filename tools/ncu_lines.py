"""Per-source-line warp-stall samples and instruction share of one ncu capture
(--import-source on): python tools/ncu_lines.py <rep> [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur, hdr, data = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        inst = int(r[hdr.index("Instructions Executed")] or 0)
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    data.append((samp, inst, cur, r[0], r[1][:100]))
ts = sum(d[0] for d in data) or 1
ti = sum(d[1] for d in data) or 1
for d in sorted(data, key=lambda x: -x[0])[:top]:
    print(f"{d[2]:>12}:{d[3]:<5} samp {d[0] / ts * 100:5.1f}% inst {d[1] / ti * 100:5.1f}%  {d[4]}")
