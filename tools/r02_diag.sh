#!/bin/bash
# round-2 first diagnostics: host info, baseline numbers, B=1 timeline, wpi A/B,
# tcgen05 wait counters at B=16/64.
O=gpurun_out/r02_diag
mkdir -p $O
{ nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > $O/host.txt 2>&1
for b in 1 4 16 64; do
  timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}.json 2>$O/b${b}.err
done
for wpi in 2 4; do
  MK_ATTN_WPI=$wpi timeout 300 python bench.py --batch 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/b1_wpi$wpi.json 2>/dev/null
done
for b in 16 64; do
  MK_DEBUG=4 timeout 300 python bench.py --batch $b --steps 5 --warmup 3 --no-cpu-baseline > $O/b${b}_dbg4.json 2>/dev/null
done
timeout 300 python tools/timeline.py --batch 1 --out $O/timeline_b1.json > $O/timeline_b1.log 2>&1
MK_ATTN_WPI=4 timeout 300 python tools/timeline.py --batch 1 --out $O/timeline_b1_wpi4.json > $O/timeline_b1_wpi4.log 2>&1
timeout 300 python tools/timeline.py --batch 64 --out $O/timeline_b64.json > $O/timeline_b64.log 2>&1
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02_diag/*.json")):
    if "timeline" in p: continue
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        c = d.get("counters_per_step", {})
        print(p.split("/")[-1], d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"),
              {k: c[k] for k in c if k.startswith("wait") or k == "mma_chunks"})
    except Exception as e:
        print(p, "FAILED", e)
PY
