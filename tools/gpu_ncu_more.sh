O=gpurun_out/final3
mkdir -p $O
for cfg in "b8:--batch 8" "b16:--batch 16"; do
  tag=${cfg%%:*}; args=${cfg#*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:megakernel -s 4 -c 1 \
    -o $O/ncu_$tag -f python bench.py $args --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full_$tag.log 2>&1
  ncu -i $O/ncu_$tag.ncu-rep --page raw --csv > $O/ncu_${tag}_raw.csv 2>/dev/null
  rm -f $O/ncu_$tag.ncu-rep
done
ls -la $O
