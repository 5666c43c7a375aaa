#!/bin/bash
O=gpurun_out/r02b_cross
mkdir -p $O
for b in 2 3; do
  timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/gemv_b$b.json 2>/dev/null
  MK_UMMA_MIN_BATCH=2 timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/umma_b$b.json 2>/dev/null
done
MK_UMMA_MIN_BATCH=1 timeout 300 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/umma_b1.json 2>/dev/null
timeout 300 python bench.py --batch 4 --steps 20 --warmup 5 --no-cpu-baseline > $O/umma_b4.json 2>/dev/null
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_cross/*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["config"]["topology"]["sms_per_die"])
    except Exception as e:
        print(p, "FAILED", e)
PY
