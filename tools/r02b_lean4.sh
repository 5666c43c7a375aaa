#!/bin/bash
O=gpurun_out/r02b_lean4
mkdir -p $O
for v in post lean4; do
  for b in 1 2 3; do
    MK_LIB_PATH=tools/ab/libmk_$v.so timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/${v}_b$b.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_lean4/*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["config"]["topology"]["sms_per_die"])
    except Exception as e:
        print(p, "FAILED", e)
PY
timeout 600 python -m pytest tests/test_gpu_megakernel.py -q -x -k "gemv or toy_decode" 2>&1 | tail -2
