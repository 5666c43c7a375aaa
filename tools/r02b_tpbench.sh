#!/bin/bash
O=gpurun_out/r02b_tpbench
mkdir -p $O
for b in 1 16; do
  timeout 600 python bench.py --tp-emulate 2 --batch $b --steps 10 --warmup 3 > $O/tp2_b$b.json 2>$O/tp2_b$b.err; tail -c 900 $O/tp2_b$b.json; tail -3 $O/tp2_b$b.err
done
timeout 300 python bench.py --steps 20 --warmup 5 > $O/b1_default.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/b1_default.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['e2e'])"
