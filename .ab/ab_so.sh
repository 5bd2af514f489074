# A/B of two library builds: .ab/libieds_<v>.so copied over the in-tree library before each run
mkdir -p gpurun_out
rm -f gpurun_out/ab_summary.txt
for v in "$@" "$@"; do
cp .ab/libieds_$v.so paper_2112_10591_b200/lib/libieds.so
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-exact --no-f3 --no-f4 --no-latency > gpurun_out/ab_$v.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), {k:(round(v['avg_ms'],4)) for k,v in d['kernels'].items()}, 'u8', round(d['f1_u8_surface']['value']), 'f16', round(d['f1_f16_surface']['value']), 'c5', round(d['c5_burst']['value']))" >> gpurun_out/ab_summary.txt
done
