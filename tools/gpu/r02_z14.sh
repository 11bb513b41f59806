mkdir -p gpurun_out/prof
ncu --set full --import-source on --clock-control none -k regex:'span_eval' -c 1 -o gpurun_out/prof/z14_trunc2d -f python bench.py --workload trunc2d --extra '' --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/z14_trunc2d.log 2>&1; echo "ncu $?"
