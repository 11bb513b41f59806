for w in trunc1d trunc2d; do
  timeout 600 python bench.py --workload $w --extra '' > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err; echo "$w ours $?"
  timeout 900 python bench.py --workload $w --impl reference --steps 3 --warmup 1 > gpurun_out/bref_$w.json 2> gpurun_out/bref_$w.err; echo "$w ref $?"
done
/usr/bin/time -v timeout 900 python bench.py --impl reference > gpurun_out/bref_cfg4.json 2> gpurun_out/bref_cfg4.err; echo "cfg4 ref $?"
/usr/bin/time -v timeout 1200 python bench.py > gpurun_out/b_full.json 2> gpurun_out/b_full.err; echo "full $?"
