#!/bin/bash
O=gpurun_out/r02b_qpre
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_qwen3_8b.py tests/test_gpu_megakernel.py tests/test_gpu_paged.py -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for b in 1 16 64; do
  timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/b${b}.json 2>$O/b${b}.err
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_qpre/b*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["roofline"]["frac"], d["config"]["topology"]["sms_per_die"])
    except Exception as e:
        print(p, "FAILED", e)
PY
timeout 300 python tools/trace_stages.py --batch 64 --out $O/trace_b64.json > $O/trace_b64.log 2>&1
grep -E "L17.attn|total" $O/trace_b64.log
