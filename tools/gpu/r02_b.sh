python -m pytest tests/test_gpu_scans.py tests/test_gpu_group.py tests/test_gpu_pipeline.py tests/test_gpu_boxfft.py -q -p no:cacheprovider > gpurun_out/pytest_b.log 2>&1; echo pytest=$?
timeout 600 python bench.py --extra '' --no-cpu-baseline > gpurun_out/b_cfg4_b.json 2> gpurun_out/b_cfg4_b.err; echo bench=$?
