"""Dump the raw die-probe latency matrix (diagnostics)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_15379_b200 import _lib as L  # noqa: E402

lib = L.load()
buf = (C.c_uint32 * (L.MAX_SMS * 512))()
n = C.c_int32()
L.check(lib.mk_probe_raw(0, buf, C.byref(n)))
a = np.frombuffer(buf, dtype=np.uint32).reshape(L.MAX_SMS, 512)[:, :n.value]
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/probe_raw.npy", a)
t = L.Topology()
L.check(lib.mk_probe(0, C.byref(t)))
print("dies", t.num_dies, list(t.sms_per_die)[:2], t.separation, t.near_cycles, t.far_cycles)
print("row means", a[:148].mean(1)[:20])
