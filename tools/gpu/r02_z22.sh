python -m pytest tests/test_gpu_stencil_cy.py tests/test_gpu_stencil.py -q -x -p no:cacheprovider > gpurun_out/pytest_z22.log 2>&1; echo pytest_z22=$?
bash tools/macro_ab.sh "--workload cfg2 --extra ''" "" "-DNLG_CY_W2=4 -DNLG_CY_MINB2=4" > gpurun_out/z22_cfg2.log 2>&1
