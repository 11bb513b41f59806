for w in cfg4b cfg2 cfg3; do bash tools/macro_ab.sh "--workload $w --extra ''" "-DNLG_CY_U=2"; done > gpurun_out/z20_u2.log 2>&1
NLG_NVCC_EXTRA="-DNLG_CY_U=2" python -m paper_1905_08375_b200.build > /dev/null 2>&1
python -m pytest tests/test_gpu_stencil_cy.py tests/test_gpu_stencil.py -q -x -p no:cacheprovider > gpurun_out/pytest_z20.log 2>&1; echo pytest_z20=$?
