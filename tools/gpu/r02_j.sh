python -m pytest tests/test_gpu_stencil.py tests/test_gpu_parity.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > gpurun_out/pytest_j.log 2>&1; echo pytest=$?
for w in cfg4b cfg2 cfg3; do timeout 600 python bench.py --workload $w --extra '' --no-cpu-baseline > gpurun_out/b_st_$w.json 2> gpurun_out/b_st_$w.err; echo "$w $?"; done
