# column-lane stencil: ring window vs shift, ncu captures
mkdir -p gpurun_out/prof
python -m pytest tests/test_gpu_stencil.py -q -x -p no:cacheprovider > gpurun_out/pytest_cy2.log 2>&1; echo pytest_cy2=$?
for w in cfg2 cfg4b; do timeout 600 python bench.py --workload $w --extra '' --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w ring', round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,3))"; done > gpurun_out/cy_ring.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:'stencil_cy' -c 1 -o gpurun_out/prof/cy_cfg2 -f python tools/prof_apply.py cfg2 4096 1 > gpurun_out/prof/cy_cfg2.log 2>&1; echo "ncu cfg2 $?"
ncu --set full --import-source on --clock-control none -k regex:'stencil_cy' -c 1 -o gpurun_out/prof/cy_cfg4b -f python tools/prof_apply.py cfg4b 256 1 > gpurun_out/prof/cy_cfg4b.log 2>&1; echo "ncu cfg4b $?"
bash tools/macro_ab.sh "--workload cfg4b --extra ''" "-DNLG_CY_RING=0" "-DNLG_CY_W3=4" "-DNLG_CY_W3=1" > gpurun_out/cy_macro_4b.log 2>&1
bash tools/macro_ab.sh "--workload cfg2 --extra ''" "-DNLG_CY_RING=0" "-DNLG_CY_W2=2" > gpurun_out/cy_macro_2.log 2>&1
