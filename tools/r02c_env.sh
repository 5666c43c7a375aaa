#!/bin/bash
# A/B of an environment knob on the current build: VAR=name VALUES="0 1" BATCHES="1 16 64"
O=gpurun_out/r02c_env; mkdir -p $O
for rep in 1 2; do for b in ${BATCHES:-1 16 64}; do for v in ${VALUES:-0 1}; do
  env $VAR=$v timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline 2>$O/err_${b}_${v}.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('B=$b $VAR=$v', d['ms_per_step'], d['config']['topology']['sms_per_die'])"
done; done; done | tee $O/env.log
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log; fi
