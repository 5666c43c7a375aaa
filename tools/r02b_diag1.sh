#!/bin/bash
# B=1 gap diagnosis: sub-phase trace, L2 prefetch depth sweep, ncu L2 hit / DRAM bytes with and without prefetch
O=gpurun_out/r02b_diag1
mkdir -p $O
timeout 300 python tools/trace_stages.py --batch 1 --out $O/trace_b1.json > $O/trace_b1.log 2>&1
MK_PREFETCH=16 timeout 300 python tools/trace_stages.py --batch 1 --out $O/trace_b1_pf16.json > $O/trace_b1_pf16.log 2>&1
for pf in 0 8 16 32 48; do
  MK_PREFETCH=$pf timeout 300 python bench.py --batch 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/b1_pf$pf.json 2>/dev/null
done
for pf in 0 16; do
  MK_PREFETCH=$pf timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum \
    --clock-control none -k regex:megakernel --launch-skip 4 -c 1 --csv \
    python bench.py --batch 1 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_b1_pf$pf.csv 2>&1
done
python - <<'PY'
import json, glob
for p in sorted(glob.glob("gpurun_out/r02b_diag1/b1_pf*.json")):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        print(p.split("/")[-1], d["ms_per_step"], d["roofline"]["frac"])
    except Exception as e:
        print(p, "FAILED", e)
PY
head -40 $O/trace_b1.log
