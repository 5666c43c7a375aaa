#!/bin/bash
O=gpurun_out/r02b_ring11
mkdir -p $O
nvidia-smi --query-gpu=name --format=csv > $O/host.txt
for b in 1 2 4 16 64; do
  timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/b${b}.json 2>$O/b${b}.err
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_ring11/b*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["roofline"]["frac"], d["config"]["topology"]["sms_per_die"])
    except Exception as e:
        print(p, "FAILED", e)
PY
timeout 300 python tools/trace_stages.py --batch 1 --out $O/trace_b1.json > $O/trace_b1.log 2>&1
grep -E "L17|lm_head|total" $O/trace_b1.log
