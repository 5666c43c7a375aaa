python - <<'PY'
import sys, os, json
sys.path.insert(0, "tools")
from umma_micro import run
for dbg in (4, 12, 28):
    gbs, ms, err, ctr = run(98304, 4096, 64, True, dbg)
    print(json.dumps(dict(debug=dbg, gbs=round(gbs, 1), waits=ctr)))
PY
