#!/bin/bash
O=gpurun_out/r02c_detail
mkdir -p $O
timeout 300 python tools/trace_stages.py --batch 16 --detail L17.o_proj --detail L17.qkv --detail L17.down --detail L17.attn_reduce --out $O/trace_b16.json > $O/trace_b16.log 2>&1
timeout 300 python tools/trace_stages.py --batch 16 --no-ksplit --detail L17.o_proj --out $O/trace_b16_noks.json > $O/trace_b16_noks.log 2>&1
timeout 300 python tools/trace_stages.py --batch 64 --detail L17.o_proj --detail L17.down --out $O/trace_b64.json > $O/trace_b64.log 2>&1
