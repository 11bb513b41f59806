mkdir -p gpurun_out/prof
#python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_stencil.py tests/test_gpu_expsum.py tests/test_gpu_reference_pins.py -q -x -p no:cacheprovider > gpurun_out/pytest_d.log 2>&1; echo pytest=$?
python tools/prof_direct.py cfg2 1024 3 > gpurun_out/prof/r02_direct_plain2.log 2>&1
python tools/prof_direct.py cfg4 256 2 >> gpurun_out/prof/r02_direct_plain2.log 2>&1
ncu --set full --import-source on --clock-control none --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
    -k regex:direct -c 1 -o gpurun_out/prof/r02b_full_direct_cfg2 -f python tools/prof_direct.py cfg2 1024 1 > gpurun_out/prof/r02b_full_direct.log 2>&1; echo "direct $?"
ncu --set full --import-source on --clock-control none -k regex:'f3_(rows|cols|zstencil|ties)' -c 6 -o gpurun_out/prof/r02b_full_cfg4 -f \
    python tools/prof_apply.py cfg4 768 1 > gpurun_out/prof/r02b_full_cfg4.log 2>&1; echo "full cfg4 $?"
