mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "workload or chunking or full_size or banded" > gpurun_out/ab_tests.log 2>&1
for v in 0 1 0 1; do
IEDS_FRAME_PREFETCH=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-exact --no-f3 --no-f4 --no-latency --no-c2 > gpurun_out/ab_$v.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print($v, round(d['value']), {k:(round(v['avg_ms'],4)) for k,v in d['kernels'].items()}, 'u8', round(d['f1_u8_surface']['value']), 'c5', round(d['c5_burst']['value']))" >> gpurun_out/ab_summary.txt
done
