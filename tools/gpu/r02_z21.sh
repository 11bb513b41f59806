python -m pytest tests/test_gpu_stencil_cy.py tests/test_gpu_stencil.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > gpurun_out/pytest_z21.log 2>&1; echo pytest_z21=$?
timeout 900 python tools/fuzz_cy.py 80 21 > gpurun_out/fuzz_z21.log 2>&1; echo fuzz=$?
for w in cfg4b cfg2; do timeout 600 python bench.py --workload $w --extra '' --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,3))"; done > gpurun_out/z21_ab.log 2>&1
