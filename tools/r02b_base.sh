#!/bin/bash
# round-2 session 2 baseline: full GPU suite, default bench line, batch sweep, B=1 trace
O=gpurun_out/r02b_base
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/host.txt 2>&1; nproc >> $O/host.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; tail -8 $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench_default.json 2>$O/bench_default.err; tail -c 600 $O/bench_default.json
for b in 2 4 8 16 32 64; do
  timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}.json 2>/dev/null
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_base/b*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["roofline"]["frac"])
    except Exception as e:
        print(p, "FAILED", e)
PY
