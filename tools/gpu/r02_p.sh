for c in 12 24 48; do
  NLG_PIPE_CHUNKS=$c timeout 300 python bench.py --extra '' --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks=$c', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e9,3))"
done > gpurun_out/chunks_ab.log 2>&1
for c in 8 16 32; do
  NLG_PIPE_CHUNKS=$c timeout 300 python bench.py --workload cfg4b --extra '' --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4b chunks=$c', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e9,3))"
done >> gpurun_out/chunks_ab.log 2>&1
python -m pytest tests/test_gpu_scans.py tests/test_gpu_parity.py tests/test_gpu_solve.py -q -x -p no:cacheprovider > gpurun_out/pytest_p.log 2>&1; echo pytest=$?
for w in trunc1d trunc2d; do timeout 300 python bench.py --workload $w --extra '' --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['roofline']['kernel_ms_per_launch'].items()})"; done >> gpurun_out/chunks_ab.log 2>&1
