# A/B of prebuilt libraries (run under gpurun): bash tools/gpu_ab.sh "<bench args>" lib1 lib2 ...
args=$1; shift
for rep in 1 2; do
for lib in "$@"; do
  MK_LIB_PATH=$lib timeout 300 python bench.py $args --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$lib', d['ms_per_step'], d['config']['topology']['sms_per_die'])"
done; done
