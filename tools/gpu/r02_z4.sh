# column-lane stencil: R = 8 defaults (exact reach, 3 CTAs / SM in 3-D), variants
python -m pytest tests/test_gpu_stencil.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py tests/test_gpu_group.py -q -x -p no:cacheprovider > gpurun_out/pytest_cy4.log 2>&1; echo pytest_cy4=$?
for w in cfg2 cfg4b; do timeout 600 python bench.py --workload $w --extra '' --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w default', round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,3))"; done > gpurun_out/cy_def4.log 2>&1
bash tools/macro_ab.sh "--workload cfg2 --extra ''" "-DNLG_CY_W2=16 -DNLG_CY_MINB2=1" "-DNLG_CY_R=12 -DNLG_CY_W2=6 -DNLG_CY_MINB2=2" "-DNLG_CY_ONEVAR=1" > gpurun_out/cy_v4_2.log 2>&1
bash tools/macro_ab.sh "--workload cfg4b --extra ''" "-DNLG_CY_ONEVAR=1" "-DNLG_CY_W3=2 -DNLG_CY_MINB3=4" "-DNLG_CY_R=12 -DNLG_CY_W3=3 -DNLG_CY_MINB3=2" > gpurun_out/cy_v4_4b.log 2>&1
