#!/bin/bash
O=gpurun_out/r02b_umma2
mkdir -p $O
timeout 300 python tools/trace_stages.py --batch 64 --detail L17.qkv --detail L17.o_proj --detail L17.down --detail L17.rms1 --out $O/trace_b64.json > $O/trace_b64.log 2>&1
grep -A40 -- "-- L17" $O/trace_b64.log
MK_DEBUG=4 timeout 300 python bench.py --batch 64 --steps 5 --warmup 3 --no-cpu-baseline > $O/b64_dbg4.json 2>/dev/null
python -c "
import json; d=json.loads(open('$O/b64_dbg4.json').read().strip().splitlines()[-1]); c=d['counters_per_step']; print(d['ms_per_step'], {k:c[k] for k in c if k.startswith('wait') or k=='mma_chunks'})"
