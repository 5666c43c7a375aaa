for b in 2 4 8; do
  for m in 16 2; do
    MK_UMMA_MIN_BATCH=$m timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B=$b umma_min=$m', d['ms_per_step'])"
  done
done
