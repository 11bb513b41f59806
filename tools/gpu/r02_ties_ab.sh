bash tools/macro_ab.sh "--extra ''" "" "-DNLG_TIES_SKIP=0" "-DNLG_TIES_MINB=3" "-DNLG_TIES_NOSUM=1" > gpurun_out/ties_ab.log 2>&1
