#!/bin/bash
# Full measurement pass (run under gpurun): default bench line, reference arm,
# batch / mode sweep, ncu launch list + one full capture.  Outputs -> gpurun_out/
set -u
mkdir -p gpurun_out/sweep
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/sweep/smi.csv
timeout 900 python bench.py > gpurun_out/sweep/bench_default.json 2> gpurun_out/sweep/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/sweep/bench_reference.json 2> gpurun_out/sweep/bench_reference.err
for b in 2 4 8 16 32 64; do
  timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sweep/b${b}_m_tile.json 2>/dev/null
done
for b in 1 32 64; do
  timeout 300 python bench.py --batch $b --steps 5 --warmup 3 --mode standard --no-cpu-baseline > gpurun_out/sweep/b${b}_standard.json 2>/dev/null
done
for m in chiplet_m_split chiplet_n_major; do
  timeout 300 python bench.py --batch 32 --steps 5 --warmup 3 --mode $m --no-cpu-baseline > gpurun_out/sweep/b32_${m}.json 2>/dev/null
done
timeout 400 python tools/timeline.py --batch 1 --out gpurun_out/sweep/timeline_b1.json > gpurun_out/sweep/timeline_b1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sweep/launches_b1.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:megakernel -s 4 -c 1 \
    -o gpurun_out/sweep/ncu_b1 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --section MemoryWorkloadAnalysis --section SpeedOfLight --clock-control none -k regex:megakernel -s 4 -c 1 \
    -o gpurun_out/sweep/ncu_b32 -f python bench.py --batch 32 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --section MemoryWorkloadAnalysis --section SpeedOfLight --clock-control none -k regex:megakernel -s 4 -c 1 \
    -o gpurun_out/sweep/ncu_b32_std -f python bench.py --batch 32 --steps 2 --warmup 3 --mode standard --no-cpu-baseline > /dev/null 2>&1
echo sweep done
