#!/bin/bash
# MMA-warp stamps (debug bit 5): stamp6 = first operand pair ready, stamp7 = last commit issued
O=gpurun_out/r02c_mma
mkdir -p $O
MK_DEBUG=32 timeout 300 python tools/trace_stages.py --batch 16 --detail L17.o_proj --detail L17.qkv --detail L17.down --out $O/trace_b16.json > $O/trace_b16.log 2>&1
MK_DEBUG=32 timeout 300 python tools/trace_stages.py --batch 16 --no-ksplit --detail L17.o_proj --out $O/trace_b16_noks.json > $O/trace_b16_noks.log 2>&1
