#!/bin/bash
# descriptor cache: tests + traces + ksplit threshold sweep + precision gap
O=gpurun_out/r02_pcache
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_qwen3_8b.py::test_qwen3_8b_36_layers_greedy_and_sync_accounting > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
for b in 1 64; do
  timeout 300 python tools/trace_stages.py --batch $b --out $O/trace_b$b.json > $O/trace_b$b.log 2>&1
done
for kb in 0.85 0.95 0.99; do
  for b in 1 4 64; do
    MK_KSPLIT_BALANCE=$kb timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}_ks$kb.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02_pcache/b*_ks*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["roofline"]["frac"])
    except Exception as e:
        print(p, "FAILED", e)
PY
timeout 900 python tools/precision_gap.py --layers 36 --tokens 6 --out $O/precision_gap_36.json 2>&1 | tail -2
timeout 600 python tools/precision_gap.py --layers 2 --tokens 6 --out $O/precision_gap_2.json 2>&1 | tail -1
