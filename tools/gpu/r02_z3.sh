# column-lane stencil: R = 8 variants
bash tools/macro_ab.sh "--workload cfg2 --extra ''" "-DNLG_CY_R=8 -DNLG_CY_RING=1 -DNLG_CY_MINB=4" "-DNLG_CY_R=8 -DNLG_CY_RING=0 -DNLG_CY_MINB=4" "-DNLG_CY_R=8 -DNLG_CY_RING=1 -DNLG_CY_MINB=2 -DNLG_CY_W2=8" > gpurun_out/cy_r8_2.log 2>&1
bash tools/macro_ab.sh "--workload cfg4b --extra ''" "-DNLG_CY_R=8 -DNLG_CY_RING=1 -DNLG_CY_MINB=4 -DNLG_CY_W3=4" "-DNLG_CY_R=8 -DNLG_CY_RING=0 -DNLG_CY_MINB=4 -DNLG_CY_W3=4" "-DNLG_CY_R=8 -DNLG_CY_RING=1 -DNLG_CY_MINB=2 -DNLG_CY_W3=8" > gpurun_out/cy_r8_4b.log 2>&1
NLG_NVCC_EXTRA="-DNLG_CY_R=8 -DNLG_CY_RING=1 -DNLG_CY_MINB=4 -DNLG_CY_W3=4" python -m paper_1905_08375_b200.build > /dev/null 2>&1
python -m pytest tests/test_gpu_stencil.py -q -x -p no:cacheprovider > gpurun_out/pytest_cy_r8.log 2>&1; echo pytest_r8=$?
