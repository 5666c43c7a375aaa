# per-stage timelines (run under gpurun):  bash tools/gpu_timeline.sh "<bench args>" tag ...
mkdir -p gpurun_out
while [ $# -ge 2 ]; do
  timeout 300 python tools/timeline.py $1 --out gpurun_out/timeline_$2.json > gpurun_out/timeline_$2.log 2>&1
  shift 2
done
