#!/bin/bash
O=gpurun_out/r02b_fold
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_qwen3_8b.py tests/test_gpu_megakernel.py -q -x -k "widths or tcgen05 or toy" > $O/pytest.log 2>&1; tail -15 $O/pytest.log
for b in 4 16 64; do
  timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/b${b}.json 2>$O/b${b}.err
  MK_NO_FOLD=1 timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/b${b}_nofold.json 2>/dev/null
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_fold/b*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["roofline"]["frac"], d["config"]["topology"]["sms_per_die"])
    except Exception as e:
        print(p, "FAILED", e)
PY
