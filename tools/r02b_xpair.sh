#!/bin/bash
O=gpurun_out/r02b_xpair
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_qwen3_8b.py tests/test_gpu_megakernel.py -q -x -k "widths or tcgen05 or toy" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for b in 3 4 16 32 64; do
  timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/b${b}.json 2>$O/b${b}.err
done
timeout 300 python bench.py --batch 64 --mode standard --steps 10 --warmup 3 --no-cpu-baseline > $O/b64_standard.json 2>/dev/null
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_xpair/b*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["roofline"]["frac"], d["config"]["topology"]["sms_per_die"])
    except Exception as e:
        print(p, "FAILED", e)
PY
