#!/bin/bash
O=gpurun_out/r02b_umma10
mkdir -p $O
python - <<'PY' 2>&1 | tee $O/umma.log
import sys, json
sys.path.insert(0, "tools")
from umma_micro import run
for (N, K) in ((98304, 4096), (24576, 4096)):
    for B in (16, 64):
        for dbg in (0, 4, 54):
            gbs, ms, err, ctr = run(N, K, B, True, dbg, check=(dbg == 0))
            print(json.dumps(dict(N=N, K=K, B=B, dbg=dbg, gbs=round(gbs, 1), err=err, waits=ctr)), flush=True)
PY
for b in 4 16 64; do
  timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}.json 2>$O/b${b}.err
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_umma10/b*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["roofline"]["frac"])
    except Exception as e:
        print(p, "FAILED", e)
PY
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
