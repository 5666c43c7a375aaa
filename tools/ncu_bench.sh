#!/bin/bash
# ncu captures of the megakernel (run under gpurun; 1 GPU).
#   tools/ncu_bench.sh <tag> <bench args...>
# -> gpurun_out/ncu_<tag>.ncu-rep (full set, 1 launch after warm-up) and
#    gpurun_out/launches_<tag>.csv (gpu__time_duration of every launch)
set -u
tag=$1; shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ncu_launch_${tag}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:megakernel -s 4 -c 1 \
    -o gpurun_out/ncu_${tag} -f \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ncu_full_${tag}.log 2>&1
echo "ncu done: $tag"
