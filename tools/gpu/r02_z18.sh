python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_group.py tests/test_gpu_stencil.py -q -x -p no:cacheprovider > gpurun_out/pytest_z18.log 2>&1; echo pytest_z18=$?
