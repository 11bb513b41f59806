#!/bin/bash
# run bench.py for each workload (no CPU baseline) and print a one-line summary each
mkdir -p gpurun_out
for w in "$@"; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>gpurun_out/b_$w.err | tail -1 > gpurun_out/b_$w.json
done
for w in "$@"; do
python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/b_{w}.json").read())
    st = d["roofline"].get("stage_ms_per_launch")
    print(w, "ms/step %.4f" % d["ms_per_step"], "value %.4g" % d["value"], "frac %.4f" % d["roofline"]["frac"],
          "e2e %.4g" % d["e2e"]["value"], "stages", st, "launches", d.get("gpu_launches"))
except Exception as e:
    print(w, "ERR", e, open(f"gpurun_out/b_{w}.err").read()[-800:])
PY
done
