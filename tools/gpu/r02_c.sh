python -m pytest tests/test_gpu_boxfft.py tests/test_gpu_pipeline.py tests/test_gpu_group.py -q -x -p no:cacheprovider > gpurun_out/pytest_c.log 2>&1; echo pytest=$?
timeout 600 python bench.py --extra '' --no-cpu-baseline > gpurun_out/b_cfg4_c.json 2> gpurun_out/b_cfg4_c.err; echo bench=$?
NLG_TIES_TMA=0 timeout 600 python bench.py --extra '' --no-cpu-baseline > gpurun_out/b_cfg4_c0.json 2> gpurun_out/b_cfg4_c0.err; echo bench0=$?
