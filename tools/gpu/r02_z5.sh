# column-lane stencils incl. peridynamics: parity, A/B, ncu
mkdir -p gpurun_out/prof
python -m pytest tests/test_gpu_stencil.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py tests/test_gpu_group.py tests/test_gpu_reference_pins.py -q -x -p no:cacheprovider > gpurun_out/pytest_cy5.log 2>&1; echo pytest_cy5=$?
for w in cfg3 cfg2 cfg4b; do for c in 1 0; do NLG_ST_CY=$c timeout 600 python bench.py --workload $w --extra '' --no-cpu-baseline 2>gpurun_out/cy5_${w}_$c.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w CY=$c', round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,3))"; done; done > gpurun_out/cy5_ab.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:'stencil_cy' -c 1 -o gpurun_out/prof/cy5_cfg2 -f python tools/prof_apply.py cfg2 4096 1 > gpurun_out/prof/cy5_cfg2.log 2>&1; echo "ncu cfg2 $?"
ncu --set full --import-source on --clock-control none -k regex:'stencil_cy' -c 1 -o gpurun_out/prof/cy5_cfg3 -f python tools/prof_apply.py cfg3 4096 1 > gpurun_out/prof/cy5_cfg3.log 2>&1; echo "ncu cfg3 $?"
ncu --set full --import-source on --clock-control none -k regex:'stencil_cy' -c 1 -o gpurun_out/prof/cy5_cfg4b -f python tools/prof_apply.py cfg4b 384 1 > gpurun_out/prof/cy5_cfg4b.log 2>&1; echo "ncu cfg4b $?"
