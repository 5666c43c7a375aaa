#!/bin/bash
O=gpurun_out/r02b_postnorm
mkdir -p $O
for b in 1 2; do
  timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/b${b}.json 2>$O/b${b}.err
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_postnorm/b*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["roofline"]["frac"])
    except Exception as e:
        print(p, "FAILED", e)
PY
timeout 300 python tools/trace_stages.py --batch 1 --out $O/trace_b1.json > $O/trace_b1.log 2>&1
grep -E "L17|lm_head|total" $O/trace_b1.log
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
