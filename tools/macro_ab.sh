#!/bin/bash
# Rebuild with each NLG_NVCC_EXTRA variant and run a bench twice (A/B of build-time macros).
#   tools/macro_ab.sh "--workload cfg4 --extra ''" "" "-DNLG_TIES_SKIP=0" ...
# The first argument is the bench.py argument string; each further one a variant.
args="$1"; shift
for v in "$@"; do
  NLG_NVCC_EXTRA="$v" python -m paper_1905_08375_b200.build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for k in 1 2; do
    eval python bench.py --steps 10 --warmup 3 --no-cpu-baseline $args 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', round(d['ms_per_step'],4), {k: round(x, 3) for k, x in d['roofline']['kernel_ms_per_launch'].items()})"
  done
done
NLG_NVCC_EXTRA="" python -m paper_1905_08375_b200.build > /dev/null 2>&1
