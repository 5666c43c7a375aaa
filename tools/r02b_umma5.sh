#!/bin/bash
O=gpurun_out/r02b_umma5
mkdir -p $O
timeout 300 python tools/trace_stages.py --batch 64 --detail L17.o_proj --detail L17.qkv --out $O/trace_b64.json > $O/trace_b64.log 2>&1
grep -A16 -- "-- L17" $O/trace_b64.log
