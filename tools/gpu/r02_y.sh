# A/B: chunked PA->PB / PD->PE (L2 chaining) and a one-cell-narrower stencil tile halo
for c in 0 4 6 8 12 0; do NLG_F3_CHUNK=$c timeout 300 python bench.py --extra '' --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CHUNK=$c', round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,3), d['gpu_launches'])"; done > gpurun_out/chunk_ab.log 2>&1
NLG_F3_CHUNK=6 python -m pytest tests/test_gpu_boxfft.py -q -x -p no:cacheprovider > gpurun_out/pytest_chunk.log 2>&1; echo pytest_chunk=$?
bash tools/macro_ab.sh "--workload cfg4b --extra ''" "" "-DNLG_ST_HPAD=1" > gpurun_out/hpad_cfg4b.log 2>&1
bash tools/macro_ab.sh "--workload cfg2 --extra ''" "-DNLG_ST_HPAD=1" > gpurun_out/hpad_cfg2.log 2>&1
NLG_NVCC_EXTRA="-DNLG_ST_HPAD=1" python -m paper_1905_08375_b200.build > /dev/null 2>&1
python -m pytest tests/test_gpu_stencil.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > gpurun_out/pytest_hpad.log 2>&1; echo pytest_hpad=$?
