timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for b in 1 4 8; do
  for m in 16 1; do
    MK_ATTN_MMA_MIN_BATCH=$m timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B=$b attn_mma_min=$m', d['ms_per_step'])"
  done
done
for b in 16 32 64; do
  timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B=$b', d['ms_per_step'], d['value'])"
done
