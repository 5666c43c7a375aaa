import sys, os
sys.path.insert(0, "tools")
from gemv_micro import run
for dbg in (0, 4, 0x800, 0x2000):
    for (N, K, tn, tk, fused) in [(98304, 4096, 16, 512, False), (6144, 4096, 16, 512, False)]:
        gbs, ms = run(N, K, 1, tn, tk, dbg, fused=fused, steps=10)
        print(hex(dbg), N, K, round(gbs, 1), round(ms * 1e3, 1), "us")
