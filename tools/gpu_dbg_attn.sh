timeout 600 python -m pytest tests -m gpu -x -q -k "tcgen05" 2>&1 | tail -3
for w in 1 2; do
  for b in 16 64; do
  MK_ATTN_WPI=$w timeout 120 python tools/timeline.py --batch $b --out gpurun_out/tl_wpi${w}_b$b.json > gpurun_out/tl_wpi${w}_b$b.log 2>&1
  echo "wpi=$w B=$b"; head -5 gpurun_out/tl_wpi${w}_b$b.log; grep -E "L1\.(attn)" gpurun_out/tl_wpi${w}_b$b.log
  done
done
