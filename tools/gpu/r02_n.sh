python -m pytest tests/test_gpu_expsum.py -q -x -p no:cacheprovider > gpurun_out/pytest_n.log 2>&1; echo pytest=$?
for v in 0 67108864 100000000; do
  for k in 1 2; do
    NLG_L2_PERSIST=$v timeout 300 python bench.py --workload cfg1 --extra '' --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['roofline']['kernel_ms_per_launch'].items()})"
  done
done > gpurun_out/l2_ab.log 2>&1
NLG_L2_PERSIST=67108864 python -m pytest tests/test_gpu_expsum.py -q -x -p no:cacheprovider > gpurun_out/pytest_n2.log 2>&1; echo pytest2=$?
bash tools/gpu/r02_m.sh
