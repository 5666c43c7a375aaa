#!/bin/bash
# per-unit phase traces + prefetch A/B + parity rerun
O=gpurun_out/r02_trace
mkdir -p $O
for b in 1 64; do
  timeout 300 python tools/trace_stages.py --batch $b --out $O/trace_b$b.json > $O/trace_b$b.log 2>&1
done
for pf in 0 16 32 64; do
  MK_PREFETCH=$pf timeout 300 python bench.py --batch 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/b1_pf$pf.json 2>/dev/null
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02_trace/b1_pf*.json")):
    d = json.loads(open(p).read().strip().splitlines()[-1])
    print(p.split("/")[-1], d["ms_per_step"])
PY
bash tools/r02_parity.sh
