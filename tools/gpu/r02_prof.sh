# r02 profiles: launch lists + full captures of every timed kernel (cfg4-A, cfg1), direct kernel fp64
mkdir -p gpurun_out/prof
R='f3_|es_|fs_|cols_|stencil|span|scan|moment|direct|pack'
for w in cfg4 cfg1; do
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$R" -c 400 --csv --log-file gpurun_out/prof/r02_launches_$w.csv \
      python bench.py --workload $w --extra '' --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof/r02_launch_$w.log 2>&1
  echo "launches $w $?"
done
ncu --set full --import-source on --clock-control none -k regex:'f3_(rows|cols|zstencil|ties)' -c 6 -o gpurun_out/prof/r02_full_cfg4 -f \
    python tools/prof_apply.py cfg4 768 1 > gpurun_out/prof/r02_full_cfg4.log 2>&1; echo "full cfg4 $?"
ncu --set full --import-source on --clock-control none -k regex:'es_tail|es_carry|es_fft|cols_|fs_rows' -s 0 -c 12 -o gpurun_out/prof/r02_full_cfg1 -f \
    python tools/prof_apply.py cfg1 4194304 1 > gpurun_out/prof/r02_full_cfg1.log 2>&1; echo "full cfg1 $?"
python tools/prof_direct.py cfg2 1024 2 > gpurun_out/prof/r02_direct_plain.log 2>&1
ncu --set full --import-source on --clock-control none --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
    -k regex:direct -c 1 -o gpurun_out/prof/r02_full_direct_cfg2 -f python tools/prof_direct.py cfg2 1024 1 > gpurun_out/prof/r02_full_direct.log 2>&1; echo "direct $?"
