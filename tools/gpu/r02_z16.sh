python -m pytest tests/test_gpu_stencil_cy.py -q -x -p no:cacheprovider > gpurun_out/pytest_z16.log 2>&1; echo pytest_z16=$?
bash tools/macro_ab.sh "--workload cfg4 --extra ''" "-DNLG_F3_COLS_MINB(C)=3" > gpurun_out/z16_cols.log 2>&1
