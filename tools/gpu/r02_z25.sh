mkdir -p gpurun_out/prof
ncu --set full --import-source on --clock-control none -k regex:'scan_lookback' -c 1 -o gpurun_out/prof/z25_scan -f python bench.py --workload trunc1d --extra '' --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/z25_scan.log 2>&1; echo "ncu $?"
