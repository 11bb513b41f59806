bash tools/macro_ab.sh "--workload cfg2 --extra ''" "" "-DNLG_R2FRAC=4" > gpurun_out/ab_cfg2.log 2>&1
bash tools/macro_ab.sh "--workload cfg3 --extra ''" "-DNLG_R2PERI=2" "-DNLG_R2PERI=8" > gpurun_out/ab_cfg3.log 2>&1
bash tools/macro_ab.sh "--workload cfg4b --extra ''" "" "-DNLG_R3FRAC=4" > gpurun_out/ab_cfg4b.log 2>&1
