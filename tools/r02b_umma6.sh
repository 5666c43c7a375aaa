#!/bin/bash
O=gpurun_out/r02b_umma6
mkdir -p $O
for b in 4 16 64; do
  timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}.json 2>$O/b${b}.err
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_umma6/b*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["roofline"]["frac"])
    except Exception as e:
        print(p, "FAILED", e)
PY
MK_DEBUG=4 timeout 300 python bench.py --batch 64 --steps 5 --warmup 3 --no-cpu-baseline > $O/b64_dbg4.json 2>/dev/null
python -c "
import json; d=json.loads(open('$O/b64_dbg4.json').read().strip().splitlines()[-1]); c=d['counters_per_step']; print(d['ms_per_step'], {k:c[k] for k in c if k.startswith('wait') or k=='mma_chunks'})"
timeout 300 python tools/trace_stages.py --batch 64 --detail L17.o_proj --out $O/trace_b64.json > $O/trace_b64.log 2>&1
grep -E "L17|lm_head|total" $O/trace_b64.log | head -12
