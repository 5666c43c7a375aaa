timeout 600 python -m pytest tests -m gpu -x -q -k "tcgen05 or smoke or attention" 2>&1 | tail -2
python - <<'PY'
import sys, os, json
sys.path.insert(0, "tools")
from umma_micro import run
for (N, K) in ((98304, 4096), (24576, 4096), (8192, 12288)):
    gbs, ms, err, ctr = run(N, K, 64, True, 0, check=True)
    print(json.dumps(dict(N=N, K=K, gbs=round(gbs, 1), err=err)))
PY
for b in 8 64; do timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B=$b', d['ms_per_step'])"; done
