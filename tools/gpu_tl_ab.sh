# timeline A/B of prebuilt libraries: bash tools/gpu_tl_ab.sh "<args>" tag1 lib1 tag2 lib2
mkdir -p gpurun_out
args=$1; shift
while [ $# -ge 2 ]; do
  MK_LIB_PATH=$2 timeout 300 python tools/timeline.py $args --out gpurun_out/tl_$1.json > gpurun_out/tl_$1.log 2>&1
  shift 2
done
