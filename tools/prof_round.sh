#!/bin/bash
# launch lists (bench command, per-launch device time) and one full capture of
# the dominant kernel(s) per workload; outputs under gpurun_out/prof/
mkdir -p gpurun_out/prof
declare -A KER=( [cfg1]="es_tail_walk" [cfg2]="stencil_rb" [cfg3]="stencil_rb" [cfg4]="f3_ties f3_zstencil" [cfg4b]="stencil_rb" [cfg0]="stencil1d" )
declare -A NSZ=( [cfg1]=4194304 [cfg2]=4096 [cfg3]=4096 [cfg4]=768 [cfg4b]=768 [cfg0]=4096 )
for w in "$@"; do
  python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof/plain_$w.json 2>&1 || { echo "plain $w failed"; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'f3_|es_|fs_|stencil|span|direct|pack|regular_fft|fft_' -c 400 --csv --log-file gpurun_out/prof/launches_$w.csv \
      python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  for k in ${KER[$w]}; do
    ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/prof/full_${w}_$k \
        python tools/prof_apply.py $w ${NSZ[$w]} 2 > /dev/null 2>&1
  done
  echo "$w done"
done
