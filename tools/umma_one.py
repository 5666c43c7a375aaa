"""One umma_micro configuration (for ncu): N K B ksplit debug."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from umma_micro import run
N, K, B, ks, dbg = (int(v) for v in sys.argv[1:6])
print(run(N, K, B, bool(ks), dbg, steps=3))
