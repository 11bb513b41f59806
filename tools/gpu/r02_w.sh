mkdir -p gpurun_out/prof
ncu --set full --import-source on --clock-control none -k regex:stencil_rb -c 1 -o gpurun_out/prof/r02w_full_cfg4b -f python tools/prof_apply.py cfg4b 768 1 > gpurun_out/prof/r02w_full_cfg4b.log 2>&1; echo "cfg4b $?"
ncu --set full --import-source on --clock-control none -k regex:stencil_rb -c 1 -o gpurun_out/prof/r02w_full_cfg3 -f python tools/prof_apply.py cfg3 4096 1 > gpurun_out/prof/r02w_full_cfg3.log 2>&1; echo "cfg3 $?"
ncu --set full --import-source on --clock-control none --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
    -k regex:direct -c 1 -o gpurun_out/prof/r02w_full_direct_cfg2 -f python tools/prof_direct.py cfg2 1024 1 > gpurun_out/prof/r02w_full_direct.log 2>&1; echo "direct $?"
