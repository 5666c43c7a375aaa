# wait-time L2 prefetch depth sweep (MK_PREFETCH slots per waiting GEMM unit)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for b in 1 8 64; do
  for pf in 0 16 48; do
    MK_PREFETCH=$pf timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B=$b pf=$pf', d['ms_per_step'])"
  done
done
