NLG_NVCC_EXTRA="-DNLG_BX2=64" python -m paper_1905_08375_b200.build > /dev/null 2>&1 || echo "build failed"
python -m pytest tests/test_gpu_stencil.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > gpurun_out/pytest_u.log 2>&1; echo pytest=$?
for k in 1 2; do timeout 300 python bench.py --workload cfg2 --extra '' --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bx64', round(d['ms_per_step'],4))"; done > gpurun_out/bx_ab.log 2>&1
NLG_NVCC_EXTRA="" python -m paper_1905_08375_b200.build > /dev/null 2>&1
for k in 1 2; do timeout 300 python bench.py --workload cfg2 --extra '' --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bx32', round(d['ms_per_step'],4))"; done >> gpurun_out/bx_ab.log 2>&1
