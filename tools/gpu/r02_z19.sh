for c in 0 6 12; do NLG_F3_CHUNK=$c timeout 300 python bench.py --extra '' --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('CHUNK=$c', round(d['ms_per_step'],3), {k:(round(v,4)) for k,v in r['kernel_ms_per_launch'].items()}, r.get('kernel_share'), d['gpu_launches'])"; done > gpurun_out/z19_chunk.log 2>&1
