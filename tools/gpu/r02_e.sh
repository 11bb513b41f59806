mkdir -p gpurun_out/prof
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_stencil.py tests/test_gpu_expsum.py tests/test_gpu_reference_pins.py tests/test_gpu_boxfft.py -q -x -p no:cacheprovider > gpurun_out/pytest_e.log 2>&1; echo pytest=$?
python tools/prof_direct.py cfg2 1024 3 > gpurun_out/prof/r02_direct_plain3.log 2>&1
python tools/prof_direct.py cfg4 256 2 >> gpurun_out/prof/r02_direct_plain3.log 2>&1
ncu --set full --import-source on --clock-control none --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
    -k regex:direct -c 1 -o gpurun_out/prof/r02c_full_direct_cfg2 -f python tools/prof_direct.py cfg2 1024 1 > gpurun_out/prof/r02c_full_direct.log 2>&1; echo "direct $?"
