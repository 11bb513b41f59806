mkdir -p gpurun_out/prof
ncu --set full --import-source on --clock-control none -k regex:stencil_rb -c 1 -o gpurun_out/prof/r02_full_cfg2 -f python tools/prof_apply.py cfg2 4096 1 > gpurun_out/prof/r02_full_cfg2.log 2>&1; echo "cfg2 $?"
ncu --set full --import-source on --clock-control none -k regex:stencil_rb -c 1 -o gpurun_out/prof/r02_full_cfg4b -f python tools/prof_apply.py cfg4b 768 1 > gpurun_out/prof/r02_full_cfg4b.log 2>&1; echo "cfg4b $?"
