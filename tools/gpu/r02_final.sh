# the driver's round-end sequence: GPU tests, smoke, default bench, reference arm
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo "pytest $?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke $?"
s=$(date +%s); timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench $? $(( $(date +%s) - s )) s"
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref $? $(( $(date +%s) - s )) s"
timeout 300 python bench.py --gpus 2 > gpurun_out/final_gpus2.log 2>&1; echo "gpus2 $?"
