python -m pytest tests/test_gpu_boxfft.py tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/pytest_i.log 2>&1; echo pytest=$?
timeout 600 python bench.py --extra '' --no-cpu-baseline > gpurun_out/b_ties2.json 2> gpurun_out/b_ties2.err; echo "b $?"
timeout 600 python bench.py --extra '' --no-cpu-baseline > gpurun_out/b_ties2b.json 2> gpurun_out/b_ties2b.err; echo "b $?"
