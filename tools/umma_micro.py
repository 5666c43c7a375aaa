"""Micro-benchmark of one tcgen05 GEMM die task per die (no dependencies).

Streams an [N, K] packed weight slab against a [B, K] activation block and
prints GB/s of weight bytes for several (N, K, B, K-split) shapes.  debug bit0
makes the consumers skip the epilogue math, bit1 makes the fetch warp skip
the weight TMA (ring slots arrive empty).
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_15379_b200 import _lib as L  # noqa: E402
from paper_2604_15379_b200.lowering import PIECE_FLOATS  # noqa: E402
from paper_2604_15379_b200.runtime import halves_topology, probe  # noqa: E402
from paper_2604_15379_b200.weights import pack_umma  # noqa: E402


def run(N, K, B, ksplit, debug=0, steps=5, check=False):
    lib = L.load()
    topo = probe(0)
    if topo.num_dies != 2:
        topo = halves_topology(topo.num_sms)
    W = min(topo.sms_per_die[0], topo.sms_per_die[1]) - 1
    w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    wp = pack_umma(w, 128, 64)
    x = torch.randn(B, K, device="cuda").to(torch.bfloat16)
    y = torch.zeros(B, N, device="cuda", dtype=torch.bfloat16)
    kpart = torch.zeros(2 * W * 2 * PIECE_FLOATS, device="cuda")
    tasks, params = [], bytearray()
    n_loc = N // 2
    tm = min(64, -(-B // 16) * 16)
    n_sub = 0
    for d in range(2):
        p = L.GemmParams()
        p.w = wp.data_ptr() + d * n_loc * K * 2
        p.x, p.y = x.data_ptr(), y.data_ptr()
        p.M, p.K, p.N = B, K, n_loc
        p.T_M, p.T_N, p.T_K = tm, 128, 64
        p.ldx, p.ldy, p.ldres = K, N, K
        p.y_col0 = d * n_loc
        p.epilogue = L.EPI_NONE
        p.traversal, p.distribution, p.xcd = L.TRAV_M_MAJOR, L.DIST_M_TILE, d
        p.tile_m = p.tile_n = -1
        p.body = L.BODY_UMMA
        p.y_cols = 1 << 30
        if ksplit:
            p.ksplit, p.tile_ctr0, p.piece_floats = 1, n_sub, PIECE_FLOATS
            p.kpart = kpart.data_ptr() + d * W * 2 * PIECE_FLOATS * 4
            n_sub += n_loc // 128
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
    g = L.GraphDesc(2, 1, 2, n_sub, 2, L.SCHED_PER_DIE, W, len(params),
                    C.cast(t_arr, C.c_void_p), C.cast(r_arr, C.c_void_p),
                    C.cast(u_arr, C.c_void_p), C.cast(b_arr, C.c_void_p),
                    C.cast(pbuf, C.c_void_p))
    h = C.c_void_p()
    L.check(lib.mk_create(0, C.byref(g), C.byref(topo), C.byref(h)))
    lib.mk_set_debug(h, debug)
    for _ in range(2):
        L.check(lib.mk_step(h, None))
    L.check(lib.mk_sync(h))
    err = None
    if check and debug == 0:
        ref = (x.float() @ w.float().t())
        err = ((y.float() - ref).abs().max() / ref.abs().max()).item()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(steps):
        L.check(lib.mk_step(h, None))
    e1.record()
    torch.cuda.synchronize()
    L.check(lib.mk_sync(h))
    ms = e0.elapsed_time(e1) / steps
    ctr = None
    if debug & 4:
        c = L.Counters()
        L.check(lib.mk_counters_get(h, C.byref(c)))
        d = c.as_dict()
        n = max(1, d["mma_chunks"])
        ctr = {k: round(d[k] / n, 1) for k in ("wait_ring_empty", "wait_mma_full", "wait_mma_x",
                                               "wait_mma_tmem", "wait_epi_done")}
        ctr["chunks_per_step"] = d["mma_chunks"] // (steps + 2)
        ctr["cycles_per_chunk_wall"] = round(ms * 1e-3 * 1.9e9 / max(1, d["mma_chunks"] / (steps + 2) / (2 * W)), 1)
    lib.mk_destroy(h)
    return N * K * 2 / (ms / 1e3) / 1e9, ms, err, ctr


if __name__ == "__main__":
    out = []
    shapes = [(24576, 4096), (8192, 12288), (98304, 4096)]
    if os.environ.get("SHAPES"):      # e.g. SHAPES=98304x4096,24576x4096
        shapes = [tuple(int(v) for v in sh.split("x")) for sh in os.environ["SHAPES"].split(",")]
    batches = [int(v) for v in os.environ.get("BATCHES", "16,64").split(",")]
    kss = [bool(int(v)) for v in os.environ.get("KSPLIT", "0,1").split(",")]
    dbgs = [int(v) for v in os.environ.get("DBG", "0,2,4").split(",")]
    for (N, K) in shapes:
        for B in batches:
            for ks in kss:
                for dbg in dbgs:
                    gbs, ms, err, ctr = run(N, K, B, ks, dbg, check=True)
                    rec = dict(N=N, K=K, B=B, ksplit=ks, debug=dbg, gbs=round(gbs, 1),
                               ms=round(ms, 4), rel_err=err, waits=ctr)
                    print(json.dumps(rec), flush=True)
                    out.append(rec)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/umma_micro.json", "w"), indent=1)
