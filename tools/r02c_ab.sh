#!/bin/bash
# A/B of prebuilt libraries at several batches (interleaved, 2 reps), then GPU tests on the current build
O=gpurun_out/r02c_ab
mkdir -p $O
for rep in 1 2; do
for b in ${BATCHES:-16 64 4}; do
for lib in "$@"; do
  MK_LIB_PATH=$lib timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('B=$b', '$lib'.split('/')[-1], d['ms_per_step'], d['config']['topology']['sms_per_die'])"
done; done; done | tee $O/ab.log
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log; fi
