#!/bin/bash
# K-split non-owner tail stamps (debug bit 8): stamp6 = accumulator ready (tile_done seen), stamp7 = pieces stored + CTA barrier
O=gpurun_out/r02c_tail
mkdir -p $O
MK_DEBUG=256 timeout 300 python tools/trace_stages.py --batch 16 --detail L17.o_proj --detail L17.down --out $O/trace_b16.json > $O/trace_b16.log 2>&1
