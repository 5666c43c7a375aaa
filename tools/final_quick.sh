#!/bin/bash
# Quick re-measure of the final code (no ncu): tests, default bench line,
# reference arm, die-aware sweep and the flat baseline at 32/64.
O=gpurun_out/final2
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for b in 1 2 4 8 16 32 64; do
  timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}_m_tile.json 2>/dev/null
done
for b in 32 64; do
  timeout 300 python bench.py --batch $b --mode standard --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}_standard.json 2>/dev/null
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/final2/*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d.get("ms_per_step"), d.get("value"), (d.get("roofline") or {}).get("frac"))
    except Exception as e:
        print(p, "FAILED", e)
PY
