#!/bin/bash
# GEMV rows per ring slot (RPW = rows / 8) at B=1 / B=2, interleaved, 2 reps
O=gpurun_out/r02c_rows; mkdir -p $O
for rep in 1 2; do for b in 1 2; do for r in 16 32 8; do
  MK_GEMV_ROWS=$r timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline 2>$O/err_${b}_${r}.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('B=$b rows=$r', d['ms_per_step'], d['config']['topology']['sms_per_die'])"
done; done; done | tee $O/rows.log
