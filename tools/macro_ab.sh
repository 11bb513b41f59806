#!/bin/bash
# Rebuild with each NLG_NVCC_EXTRA variant and run the default bench twice (A/B of build-time macros).
for v in "$@"; do
  NLG_NVCC_EXTRA="$v" python -m paper_1905_08375_b200.build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for k in 1 2; do
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', round(d['ms_per_step'],4), d['config']['exp_terms'])"
  done
done
