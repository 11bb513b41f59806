for v in "-DNLG_CY_NOPF" "-DNLG_CY_HSOLD" "-DNLG_CY_NOPF -DNLG_CY_HSOLD"; do
NLG_NVCC_EXTRA="$v" python -m paper_1905_08375_b200.build > /dev/null 2>&1
echo "== $v"; python -m pytest tests/test_gpu_stencil.py -q -x -p no:cacheprovider 2>&1 | tail -2
done > gpurun_out/bisect6.log 2>&1
