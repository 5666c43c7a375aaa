"""Micro-benchmark of the GEMM die task alone (no dependencies).

One die task per die streams an [N, K] weight slab through the ring; prints
GB/s for: full, consumers-skip-math (debug 1: TMA stream rate), and
no-TMA (debug 2: consumer compute rate).
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_15379_b200 import _lib as L  # noqa: E402
from paper_2604_15379_b200.runtime import probe, halves_topology  # noqa: E402


def run(N, K, B, t_n, t_k, debug, steps=5, fused=False):
    lib = L.load()
    topo = probe(0)
    if topo.num_dies != 2:
        topo = halves_topology(topo.num_sms)
    W = min(topo.sms_per_die[0], topo.sms_per_die[1]) - 1
    dev = "cuda"
    w = torch.randn(N, K, device=dev).to(torch.bfloat16)
    x = torch.randn(B, K, device=dev).to(torch.bfloat16)
    y = torch.zeros(B, N // (2 if fused else 1), device=dev, dtype=torch.bfloat16)
    tasks, params = [], bytearray()
    n_loc = N // 2
    for d in range(2):
        p = L.GemmParams()
        p.w = w.data_ptr() + d * n_loc * K * 2
        p.x, p.y = x.data_ptr(), y.data_ptr()
        p.M, p.K, p.N = B, K, n_loc
        p.T_M, p.T_N, p.T_K = 16, t_n, t_k
        p.ldx, p.ldy, p.ldres = K, y.shape[1], K
        p.y_col0 = d * (n_loc // 2 if fused else n_loc)
        p.epilogue = L.EPI_SILU if fused else L.EPI_NONE
        p.traversal, p.distribution, p.xcd = L.TRAV_M_MAJOR, L.DIST_M_TILE, d
        p.tile_m = p.tile_n = -1
        p.stage_x = 1 if min(16, B) * K * 2 <= 32768 else 0
        t = L.Task(); t.op = L.OP_GEMM; t.level = L.LEVEL_CHIPLET; t.die = d
        t.wait0 = t.wait1 = -1; t.signal = 0; t.n_units = 1; t.sub_ctr = -1
        t.param_off = len(params); t.graph_index = -1
        params += bytes(p)
        tasks.append(t)
    t_arr = (L.Task * 2)(*tasks)
    u_arr = (L.Unit * 2)(L.Unit(0, 0, 0, 0), L.Unit(1, 0, 0, 0))
    b_arr = (C.c_int32 * 3)(0, 1, 2)
    r_arr = (C.c_int32 * 1)(2)
    pbuf = C.create_string_buffer(bytes(params), len(params))
    g = L.GraphDesc(2, 1, 2, 0, 2, L.SCHED_PER_DIE, W, len(params),
                    C.cast(t_arr, C.c_void_p), C.cast(r_arr, C.c_void_p),
                    C.cast(u_arr, C.c_void_p), C.cast(b_arr, C.c_void_p),
                    C.cast(pbuf, C.c_void_p))
    h = C.c_void_p()
    L.check(lib.mk_create(0, C.byref(g), C.byref(topo), C.byref(h)))
    lib.mk_set_debug(h, debug)
    for _ in range(2):
        L.check(lib.mk_step(h, None))
    L.check(lib.mk_sync(h))
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(steps):
        L.check(lib.mk_step(h, None))
    e1.record()
    torch.cuda.synchronize()
    L.check(lib.mk_sync(h))
    ms = e0.elapsed_time(e1) / steps
    lib.mk_destroy(h)
    return N * K * 2 / (ms / 1e3) / 1e9, ms


if __name__ == "__main__":
    out = []
    for (N, K, B, tn, tk, fused) in [(24576, 4096, 1, 8, 512, True), (98304, 4096, 1, 8, 1024, False), (98304, 12288, 1, 16, 512, False),
                                      (98304, 4096, 1, 16, 512, False), (98304, 4096, 1, 32, 256, False),
                                      (98304, 4096, 4, 16, 512, False), (98304, 4096, 8, 32, 256, False)]:
        for dbg in (0, 1, 2):
            gbs, ms = run(N, K, B, tn, tk, dbg, fused=fused)
            rec = dict(N=N, K=K, B=B, tile=(tn, tk), fused=fused, debug=dbg, gbs=round(gbs, 1), ms=round(ms, 4))
            print(json.dumps(rec), flush=True)
            out.append(rec)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/gemv_micro.json", "w"), indent=1)
