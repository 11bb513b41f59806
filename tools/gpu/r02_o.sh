for c in 4 2; do for k in 1 2; do
  NLG_F3_COLS=$c timeout 300 python bench.py --extra '' --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cols=$c', round(d['ms_per_step'],4), {k: round(x,3) for k,x in d['roofline']['kernel_ms_per_launch'].items()})"
done; done > gpurun_out/cols_ab.log 2>&1
NLG_F3_COLS=2 python -m pytest tests/test_gpu_boxfft.py -q -x -p no:cacheprovider > gpurun_out/pytest_o.log 2>&1; echo pytest=$?
