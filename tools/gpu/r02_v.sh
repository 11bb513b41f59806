NLG_NVCC_EXTRA="-DNLG_BX3=64" python -m paper_1905_08375_b200.build > /dev/null 2>&1 || echo "build failed"
python -m pytest tests/test_gpu_stencil.py -q -x -p no:cacheprovider -k "3" > gpurun_out/pytest_v.log 2>&1; echo pytest=$?
for k in 1 2; do timeout 300 python bench.py --workload cfg4b --extra '' --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bx3=64', round(d['ms_per_step'],4))"; done > gpurun_out/bx3_ab.log 2>&1
NLG_NVCC_EXTRA="" python -m paper_1905_08375_b200.build > /dev/null 2>&1
