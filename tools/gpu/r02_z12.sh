# final-state validation + profiles of the column-lane stencils (compile-time pitch build)
mkdir -p gpurun_out/prof
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/z12_pytest.log 2>&1; echo "pytest $?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z12_smoke.log 2>&1; echo "smoke $?"
s=$(date +%s); timeout 1500 python bench.py > gpurun_out/z12_bench.json 2> gpurun_out/z12_bench.err; echo "bench $? $(( $(date +%s) - s )) s"
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/z12_bench_ref.json 2> gpurun_out/z12_bench_ref.err; echo "ref $? $(( $(date +%s) - s )) s"
for w in cfg2 cfg3 cfg4b; do
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:stencil -c 60 --csv --log-file gpurun_out/prof/r02z_launches_$w.csv \
      python bench.py --workload $w --extra '' --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof/r02z_launch_$w.log 2>&1
  echo "launches $w $?"
done
ncu --set full --import-source on --clock-control none -k regex:'stencil_cy' -c 1 -o gpurun_out/prof/r02z_full_cfg2 -f python tools/prof_apply.py cfg2 4096 1 > gpurun_out/prof/r02z_full_cfg2.log 2>&1; echo "full cfg2 $?"
ncu --set full --import-source on --clock-control none -k regex:'stencil_cy' -c 1 -o gpurun_out/prof/r02z_full_cfg3 -f python tools/prof_apply.py cfg3 4096 1 > gpurun_out/prof/r02z_full_cfg3.log 2>&1; echo "full cfg3 $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:'stencil_cy' -c 1 -o gpurun_out/prof/r02z_full_cfg4b -f python tools/prof_apply.py cfg4b 768 1 > gpurun_out/prof/r02z_full_cfg4b.log 2>&1; echo "full cfg4b $?"
