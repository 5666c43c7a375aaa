#!/bin/bash
O=gpurun_out/r02b_ab5
mkdir -p $O
# guard: a step that cannot start would hit the 10 s watchdog -> keep the runs short
MK_LIB_PATH=tools/ab/libmk_regs.so timeout 120 python bench.py --batch 16 --steps 3 --warmup 3 --no-cpu-baseline > $O/probe.json 2>$O/probe.err; echo "probe rc $?"; tail -2 $O/probe.err
for rep in 1 2; do
  for v in base regs; do
    for b in 4 16 64; do
      MK_LIB_PATH=tools/ab/libmk_$v.so timeout 120 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > $O/${v}_b${b}_r$rep.json 2>/dev/null
    done
  done
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_ab5/*_r*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["config"]["topology"]["sms_per_die"])
    except Exception as e:
        print(p, "FAILED", e)
PY
