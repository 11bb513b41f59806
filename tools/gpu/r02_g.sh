python -m pytest tests/test_gpu_scans.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_g.log 2>&1; echo pytest=$?
timeout 600 python bench.py --workload trunc1d --extra '' > gpurun_out/b_trunc1d.json 2> gpurun_out/b_trunc1d.err; echo "trunc1d $?"
NLG_F3_PERS=1 timeout 600 python bench.py --extra '' --no-cpu-baseline > gpurun_out/b_pers.json 2> gpurun_out/b_pers.err; echo "pers $?"
NLG_F3_PERS=1 NLG_F3_PERS_CTAS=1 timeout 600 python bench.py --extra '' --no-cpu-baseline > gpurun_out/b_pers1.json 2> gpurun_out/b_pers1.err; echo "pers1 $?"
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bref_cfg4.json 2> gpurun_out/bref_cfg4.err; echo "cfg4 ref $? $(( $(date +%s) - s )) s"
s=$(date +%s); timeout 1200 python bench.py > gpurun_out/b_full.json 2> gpurun_out/b_full.err; echo "full $? $(( $(date +%s) - s )) s"
