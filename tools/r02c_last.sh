#!/bin/bash
# Last check of the final build: GPU suite, smoke, default bench line, batch sweep
O=gpurun_out/r02c_last; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.csv
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for b in 1 2 4 8 16 32 64; do
  timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}_m_tile.json 2>/dev/null
done
for b in 8 64; do
  timeout 300 python bench.py --batch $b --mode standard --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}_standard.json 2>/dev/null
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02c_last/*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d.get("ms_per_step"), d.get("value"), (d.get("roofline") or {}).get("frac"), d["config"]["topology"]["sms_per_die"], (d.get("e2e") or {}).get("value"))
    except Exception as e:
        print(p, "FAILED", e)
PY
