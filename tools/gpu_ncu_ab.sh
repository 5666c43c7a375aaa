# ncu A/B of prebuilt libraries on one bench config (run under gpurun):
#   bash tools/gpu_ncu_ab.sh "<bench args>" tag1 lib1 tag2 lib2 ...
mkdir -p gpurun_out
args=$1; shift
while [ $# -ge 2 ]; do
  MK_LIB_PATH=$2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:megakernel -s 4 -c 1 \
    -o gpurun_out/ncu_$1 -f python bench.py $args --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$1.log 2>&1
  shift 2
done
