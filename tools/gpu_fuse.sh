timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for b in 1 64; do
  timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B=$b', d['ms_per_step'])"
done
