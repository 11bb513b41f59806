"""Instruction mix of the densest DFMA loop of one kernel in a cubin/object.

usage: python tools/sass_loop.py <obj> <mangled-name-substring>
"""
import re
import subprocess
import sys
from collections import Counter


def main(obj, pat):
    names = subprocess.run(["cuobjdump", "-symbols", obj], capture_output=True, text=True).stdout
    fun = [w for w in re.findall(r"(_Z\S+)", names) if pat in w]
    for f in sorted(set(fun)):
        sass = subprocess.run(["cuobjdump", "-sass", "-fun", f, obj], capture_output=True, text=True).stdout
        ins = []
        for line in sass.split("\n"):
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2)))
        best = None
        for a, t in ins:
            m = re.search(r"BRA(?:\.U)? (?:!?U?P\d, )?0x([0-9a-f]+)", t)
            if m and int(m.group(1), 16) < a:
                body = [x for x in ins if int(m.group(1), 16) <= x[0] <= a]
                nd = sum("DFMA" in x[1] for x in body)
                key = (nd >= 8, nd / len(body))
                if best is None or key > best[2]:
                    best = (nd, body, key)
        if not best:
            continue
        c = Counter(re.sub(r"^@!?U?P\w+\s+", "", x[1]).split()[0].split(".")[0] for x in best[1])
        print(f[-60:], "DFMA", best[0], "total", len(best[1]), dict(c.most_common()))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
