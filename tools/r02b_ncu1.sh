#!/bin/bash
O=gpurun_out/r02b_ncu1
mkdir -p $O
MK_DEBUG=2 timeout 300 python tools/trace_stages.py --batch 1 --out $O/trace_b1_notma.json > $O/trace_b1_notma.log 2>&1
grep -E "L17|lm_head|total" $O/trace_b1_notma.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:megakernel -s 3 -c 1 \
  -o $O/b1 python bench.py --batch 1 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_b1.log 2>&1
tail -2 $O/ncu_b1.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:megakernel -s 3 -c 1 \
  -o $O/b64 python bench.py --batch 64 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_b64.log 2>&1
tail -2 $O/ncu_b64.log
