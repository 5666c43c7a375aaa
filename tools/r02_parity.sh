#!/bin/bash
# round-2: parity at the benched configuration + the whole GPU suite
O=gpurun_out/r02_parity
mkdir -p $O
MK_PARITY_OUT=$O timeout 1500 python -m pytest tests/test_gpu_qwen3_8b.py -x -q -m gpu -rA > $O/pytest_qwen.log 2>&1; tail -15 $O/pytest_qwen.log
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_gpu_qwen3_8b.py > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02_parity/*.json")):
    d = json.load(open(p))
    if "steps" in d:
        print(d["tag"], "max normwise", round(max(s["normwise_err"] for s in d["steps"]), 5),
              "max row-L2", round(max(s["row_l2_err"] for s in d["steps"]), 5), "ties", d["ties"])
    else:
        print(p, d)
PY
