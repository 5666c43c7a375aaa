#!/bin/bash
O=gpurun_out/r02b_diag2
mkdir -p $O
timeout 120 ./tools/handoff_micro > $O/handoff.txt 2>&1; cat $O/handoff.txt
for kb in 0.9 0.95 0.99; do
  MK_KSPLIT_BALANCE=$kb timeout 300 python bench.py --batch 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/b1_ks$kb.json 2>/dev/null
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_diag2/b*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["roofline"]["frac"])
    except Exception as e:
        print(p, "FAILED", e)
PY
