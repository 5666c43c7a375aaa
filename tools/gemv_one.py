"""One gemv_micro configuration (for ncu): python tools/gemv_one.py N K B t_n t_k fused debug"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemv_micro import run  # noqa: E402

N, K, B, tn, tk, fused, dbg = (int(v) for v in sys.argv[1:8])
print(run(N, K, B, tn, tk, dbg, steps=3, fused=bool(fused)))
