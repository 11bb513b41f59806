python -m pytest tests/test_gpu_boxfft.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > gpurun_out/pytest_h.log 2>&1; echo pytest=$?
timeout 600 python bench.py --extra '' --no-cpu-baseline > gpurun_out/b_pa.json 2> gpurun_out/b_pa.err; echo "pa $?"
NLG_PA_MULTI=0 timeout 600 python bench.py --extra '' --no-cpu-baseline > gpurun_out/b_pa0.json 2> gpurun_out/b_pa0.err; echo "pa0 $?"
