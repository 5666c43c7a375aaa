#!/bin/bash
O=gpurun_out/r02b_tr
mkdir -p $O
for b in 16 64; do
timeout 300 python tools/trace_stages.py --batch $b --detail L17.qkv --detail L17.down --out $O/trace_b$b.json > $O/trace_b$b.log 2>&1
grep -E "L17|lm_head|total|final|argmax" $O/trace_b$b.log | head -30
done
