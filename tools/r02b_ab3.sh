#!/bin/bash
O=gpurun_out/r02b_ab4
mkdir -p $O
for rep in 1 2; do
  for v in base regs; do
    for b in 4 16 32 64; do
      MK_LIB_PATH=tools/ab/libmk_$v.so timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/${v}_b${b}_r$rep.json 2>/dev/null
    done
  done
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_ab4/*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["config"]["topology"]["sms_per_die"])
    except Exception as e:
        print(p, "FAILED", e)
PY
MK_LIB_PATH=tools/ab/libmk_regs.so timeout 900 python -m pytest tests/test_gpu_qwen3_8b.py -q -x -k "widths" 2>&1 | tail -2
