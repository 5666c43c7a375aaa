#!/bin/bash
O=gpurun_out/r02b_b2
mkdir -p $O
for b in 1 2; do
timeout 300 python tools/trace_stages.py --batch $b --out $O/trace_b$b.json > $O/trace_b$b.log 2>&1
grep -E "L17|lm_head|total" $O/trace_b$b.log
done
