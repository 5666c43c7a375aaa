#!/bin/bash
# isolate the tcgen05 chunk-rate limiter: one die task per die, flags:
# 0 normal, 2 no weight TMA, 16 no activation TMA, 18 neither, 8 no MMA, 4 wait counters
O=gpurun_out/r02b_umma_flags
mkdir -p $O
python - <<'PY' > $O/umma_flags.log 2>&1
import sys, json
sys.path.insert(0, "tools")
from umma_micro import run
for (N, K) in ((98304, 4096), (24576, 4096)):
    for B in (16, 64):
        for dbg in (0, 2, 16, 18, 8, 4):
            gbs, ms, err, ctr = run(N, K, B, True, dbg, check=(dbg == 0))
            print(json.dumps(dict(N=N, K=K, B=B, dbg=dbg, gbs=round(gbs, 1), ms=round(ms, 4), err=err, waits=ctr)), flush=True)
PY
cat $O/umma_flags.log
