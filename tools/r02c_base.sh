#!/bin/bash
# Re-entry check on the restored code: GPU tests, smoke, default bench, batch sweep.
O=gpurun_out/r02c_base
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for b in 1 2 4 16 64; do
  timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}.json 2>/dev/null
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02c_base/*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d.get("ms_per_step"), d.get("value"), (d.get("roofline") or {}).get("frac"), d["config"].get("topology", {}).get("sms_per_die"))
    except Exception as e:
        print(p, "FAILED", e)
PY
