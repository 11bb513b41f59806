mkdir -p gpurun_out/prof
R='f3_|es_|fs_|cols_|stencil|span|scan|moment|direct|pack'
for spec in "cfg4 768 3" "cfg4b 768 2" "cfg2 4096 3" "cfg3 4096 3" "cfg0 4096 3"; do
  set -- $spec
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$R" -c 400 --csv --log-file gpurun_out/prof/r02_launches_$1.csv \
      python tools/prof_apply.py $1 $2 $3 > gpurun_out/prof/r02_launch_$1.log 2>&1
  echo "launches $1 $?"
done
