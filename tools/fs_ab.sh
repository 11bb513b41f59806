#!/bin/bash
# per-kernel device times of the cfg1 apply under ncu, for NLG_FS_PERSIST=1/0
for v in 1 0; do
  NLG_FS_PERSIST=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:'fs_|es_' -c 40 --csv --log-file gpurun_out/prof/fs_$v.csv python tools/prof_apply.py cfg1 4194304 2 > /dev/null 2>&1
done
