python -m pytest tests/test_gpu_scans.py tests/test_gpu_pipeline.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_scans.log 2>&1; echo pytest=$?
timeout 600 ncu --set full --import-source on -k regex:f3_ties -c 1 -o gpurun_out/r02_cfg4_ties -f python bench.py --extra '' --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_ties.log 2>&1; echo ncu=$?
