#!/bin/bash
# ncu full set + source counters at B=1 (stall reasons per source line) and
# the tcgen05 flag experiment
O=gpurun_out/r02_ncu
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:megakernel -s 3 -c 1 \
  -o $O/b1 python bench.py --batch 1 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_b1.log 2>&1
tail -3 $O/ncu_b1.log
bash tools/r02_umma.sh
