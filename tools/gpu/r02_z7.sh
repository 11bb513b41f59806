# column-lane stencils: variants after the even-column fix
python -m pytest tests/test_gpu_stencil.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_cy7.log 2>&1; echo pytest_cy7=$?
bash tools/macro_ab.sh "--workload cfg3 --extra ''" "" "-DNLG_CYP_MINB=4" "-DNLG_CYP_W=8 -DNLG_CYP_MINB=2" > gpurun_out/cy7_cfg3.log 2>&1
bash tools/macro_ab.sh "--workload cfg4b --extra ''" "-DNLG_CY_W3=6 -DNLG_CY_MINB3=2" "-DNLG_CY_R=12 -DNLG_CY_W3=4 -DNLG_CY_MINB3=2" > gpurun_out/cy7_cfg4b.log 2>&1
bash tools/macro_ab.sh "--workload cfg2 --extra ''" "-DNLG_CY_R=12 -DNLG_CY_W2=6 -DNLG_CY_MINB2=2" "-DNLG_CY_W2=16 -DNLG_CY_MINB2=1" > gpurun_out/cy7_cfg2.log 2>&1
