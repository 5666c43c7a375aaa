#!/bin/bash
# Per-stage phase breakdown at the batch sizes the tcgen05 body runs (and B=1 for reference).
O=gpurun_out/r02c_trace
mkdir -p $O
for b in 1 16 64; do
  timeout 300 python tools/trace_stages.py --batch $b --out $O/trace_b$b.json > $O/trace_b$b.log 2>&1
done
MK_DEBUG=4 timeout 300 python bench.py --batch 16 --steps 10 --warmup 3 --no-cpu-baseline > $O/b16_prof.json 2>$O/b16_prof.err
MK_DEBUG=4 timeout 300 python bench.py --batch 64 --steps 10 --warmup 3 --no-cpu-baseline > $O/b64_prof.json 2>$O/b64_prof.err
tail -40 $O/trace_b16.log
