#!/bin/bash
O=gpurun_out/r02b_ab6
mkdir -p $O
for rep in 1 2; do
  for v in a b; do
    for b in 1 2; do
      MK_LIB_PATH=tools/ab/libmk_$v.so timeout 120 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/${v}_b${b}_r$rep.json 2>/dev/null
    done
  done
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_ab6/*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["config"]["topology"]["sms_per_die"])
    except Exception as e:
        print(p, "FAILED", e)
PY
MK_LIB_PATH=tools/ab/libmk_b.so timeout 600 python -m pytest tests/test_gpu_megakernel.py -q -x -k "gemv or toy_decode" 2>&1 | tail -2
