#!/bin/bash
O=gpurun_out/r02b_umma13
mkdir -p $O
python - <<'PY' 2>&1 | tee $O/umma.log
import sys, json
sys.path.insert(0, "tools")
from umma_micro import run
for (N, K) in ((98304, 4096),):
    for B in (16, 64):
        for dbg in (0, 4, 54):
            gbs, ms, err, ctr = run(N, K, B, True, dbg, check=(dbg == 0))
            print(json.dumps(dict(N=N, K=K, B=B, dbg=dbg, gbs=round(gbs, 1), err=err, waits=ctr)), flush=True)
PY
