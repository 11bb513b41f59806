mkdir -p gpurun_out/prof
ncu --set full --import-source on --clock-control none -k regex:'f3_ties' -c 1 -o gpurun_out/prof/r02q_ties -f python tools/prof_apply.py cfg4 768 1 > gpurun_out/prof/r02q_ties.log 2>&1; echo "ties $?"
