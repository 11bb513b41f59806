python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_reference_pins.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > gpurun_out/pytest_t.log 2>&1; echo pytest=$?
python tools/prof_direct.py cfg2 1024 3 > gpurun_out/direct_t.log 2>&1
python tools/prof_direct.py cfg4 256 2 >> gpurun_out/direct_t.log 2>&1
python tools/prof_direct.py cfg1 262144 2 >> gpurun_out/direct_t.log 2>&1
