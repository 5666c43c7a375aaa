# GPU parity tests + a bench sweep (run under gpurun).  Usage:
#   bash tools/gpu_check.sh [pytest -k expr] -- [batches...]
mkdir -p gpurun_out
K=${1:-}
shift || true
[ "${1:-}" = "--" ] && shift
if [ -n "$K" ] && [ "$K" != "none" ]; then
  if [ "$K" = "all" ]; then timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  else timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; fi
  tail -30 gpurun_out/pytest_gpu.log
fi
for b in "$@"; do
  timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_b$b.json 2> gpurun_out/bench_b$b.err
  python -c "
import json,sys
try:
  d=json.load(open('gpurun_out/bench_b$b.json'))
  print('B=$b', d['ms_per_step'], 'ms', d['value'], 'tok/s frac', d['roofline']['frac'])
except Exception as e:
  print('B=$b failed', e); print(open('gpurun_out/bench_b$b.err').read()[-2000:])
"
done
