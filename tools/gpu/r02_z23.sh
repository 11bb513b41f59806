bash tools/macro_ab.sh "--workload cfg4 --extra ''" "-DNLG_F3_ROWS_MINB=9" "-DNLG_F3_ROWS_MINB=8" > gpurun_out/z23_rows.log 2>&1
