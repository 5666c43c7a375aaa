# bench lines for several argument sets (run under gpurun):
#   bash tools/gpu_bench_modes.sh "<bench args>" tag ...
mkdir -p gpurun_out
while [ $# -ge 2 ]; do
  timeout 300 python bench.py $1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bm_$2.json 2> gpurun_out/bm_$2.err
  python -c "
import json
try:
  d=json.load(open('gpurun_out/bm_$2.json'))
  print('$2', d['ms_per_step'], 'ms', d['value'], 'tok/s frac', d['roofline']['frac'])
except Exception as e:
  print('$2 failed', e); print(open('gpurun_out/bm_$2.err').read()[-1500:])
"
  shift 2
done
