# L2 prefetch depth sweep at B=1 (CUDA-core instance), plus parity tests
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for pf in 0 16 32 64 128; do
  MK_PREFETCH=$pf timeout 300 python bench.py --batch 1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B=1 pf=$pf', d['ms_per_step'])"
done
MK_PREFETCH=64 timeout 300 python bench.py --batch 2 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B=2 pf=64', d['ms_per_step'])"
