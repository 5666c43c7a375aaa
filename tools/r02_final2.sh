#!/bin/bash
# Round-2 measurement pass (1 GPU): GPU suite, default bench line + reference
# arm, die-aware sweep, flat baseline, ablations, TP emulation, ncu launch
# list, full-set captures (B=1, B=64), L2 / DRAM metrics for every mode.
set -u
O=gpurun_out/${OUT:-r02_final2}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $O/smi.csv 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 400 $O/bench_default.json; echo
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
run() {  # tag, args
  local tag=$1; shift
  timeout 300 python bench.py "$@" --steps 10 --warmup 3 --no-cpu-baseline > $O/$tag.json 2> $O/$tag.err
  python -c "
import json
try:
  d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]); print('$tag', d['ms_per_step'], 'ms', d['value'], 'tok/s', 'frac', d['roofline'].get('frac'))
except Exception as e: print('$tag FAILED', e)"
}
for b in 1 2 3 4 8 16 32 64; do run b${b}_m_tile --batch $b; done
MK_FUSE_ATTN_REDUCE=1 run b1_fused_reduce --batch 1
MK_FUSE_ATTN_REDUCE=1 run b16_fused_reduce --batch 16
for b in 1 8 16 32 64; do run b${b}_standard --batch $b --mode standard; done
for b in 32 64; do
  run b${b}_m_split --batch $b --mode chiplet_m_split
  run b${b}_n_major --batch $b --mode chiplet_n_major
  run b${b}_m_tile_tm16 --batch $b --t-m 16
  run b${b}_m_tile_noks --batch $b --no-ksplit
done
for b in 1 16; do run tp2emu_b${b} --batch $b --tp-emulate 2; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_b1.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch_b1.log 2>&1
for cfg in "b1:--batch 1" "b64:--batch 64"; do
  tag=${cfg%%:*}; args=${cfg#*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:megakernel -s 4 -c 1 \
    -o $O/ncu_$tag -f python bench.py $args --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full_$tag.log 2>&1
  ncu -i $O/ncu_$tag.ncu-rep --page raw --csv > $O/ncu_${tag}_raw.csv 2>/dev/null
  ncu -i $O/ncu_$tag.ncu-rep --page details --csv > $O/ncu_${tag}_details.csv 2>/dev/null
  ncu -i $O/ncu_$tag.ncu-rep --page source --csv --print-source cuda,sass > $O/ncu_${tag}_source.csv 2>/dev/null
  gzip -f $O/ncu_${tag}_source.csv
  rm -f $O/ncu_$tag.ncu-rep
done
for cfg in "b32_m_tile:--batch 32" "b32_standard:--batch 32 --mode standard" \
           "b32_m_split:--batch 32 --mode chiplet_m_split" "b32_n_major:--batch 32 --mode chiplet_n_major" \
           "b64_m_tile:--batch 64" "b64_standard:--batch 64 --mode standard" \
           "b64_m_split:--batch 64 --mode chiplet_m_split" "b64_n_major:--batch 64 --mode chiplet_n_major" \
           "b64_m_tile_tm16:--batch 64 --t-m 16" "b64_standard_tm16:--batch 64 --t-m 16 --mode standard" \
           "b16_m_tile:--batch 16" "b16_standard:--batch 16 --mode standard" \
           "b1_m_tile:--batch 1" "b1_standard:--batch 1 --mode standard"; do
  tag=${cfg%%:*}; args=${cfg#*:}
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_lookup_hit.sum,lts__t_sectors_lookup_miss.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:megakernel -s 4 -c 1 --csv python bench.py $args --steps 2 --warmup 3 --no-cpu-baseline \
    > $O/l2_$tag.csv 2> $O/l2_$tag.err
done
echo done
