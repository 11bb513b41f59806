python -m pytest tests/test_gpu_stencil_cy.py -q -x -p no:cacheprovider > gpurun_out/pytest_cy9.log 2>&1; echo pytest_cy9=$?
bash tools/macro_ab.sh "--workload cfg4b --extra ''" "-DNLG_CY_STEPSEL=1" > gpurun_out/cy9_cfg4b.log 2>&1
bash tools/macro_ab.sh "--workload cfg2 --extra ''" "-DNLG_CY_STEPSEL=1" > gpurun_out/cy9_cfg2.log 2>&1
NLG_NVCC_EXTRA="-DNLG_CY_STEPSEL=1" python -m paper_1905_08375_b200.build > /dev/null 2>&1
python -m pytest tests/test_gpu_stencil_cy.py tests/test_gpu_stencil.py -q -x -p no:cacheprovider > gpurun_out/pytest_cy9s.log 2>&1; echo pytest_cy9s=$?
