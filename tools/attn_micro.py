"""Attention-only micro-benchmark: kv_heads ATTN_PARTIAL tasks (+ optional
reduce), no dependencies, Qwen3-8B head shapes, batch B, ctx T.
Prints us per launch."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_15379_b200 import _lib as L  # noqa: E402
from paper_2604_15379_b200.runtime import probe, halves_topology  # noqa: E402
from paper_2604_15379_b200.weights import rope_tables  # noqa: E402


def run(B=1, T=1024, units=19, sub=2, reduce=False, steps=20, debug=0, log=False):
    lib = L.load()
    topo = probe(0)
    if topo.num_dies != 2:
        topo = halves_topology(topo.num_sms)
    W = min(topo.sms_per_die[0], topo.sms_per_die[1]) - 1
    QH, KVH, HD = 32, 8, 128
    G = QH // KVH
    split = 64
    t_max = T + 64
    n_splits = (t_max + split - 1) // split
    dev = "cuda"
    qkv = torch.randn(B, (QH + 2 * KVH) * HD, device=dev).to(torch.bfloat16)
    kc = torch.randn(B, KVH, t_max, HD, device=dev).to(torch.bfloat16)
    vc = torch.randn(B, KVH, t_max, HD, device=dev).to(torch.bfloat16)
    g = torch.ones(HD, device=dev, dtype=torch.bfloat16)
    cos, sin = rope_tables(HD, 1e6, t_max)
    cos, sin = cos.to(dev), sin.to(dev)
    pos = torch.full((B,), T, device=dev, dtype=torch.int32)
    part = torch.zeros(B * KVH * n_splits * 8 * (HD + 4), device=dev)
    out = torch.zeros(B, QH * HD, device=dev, dtype=torch.bfloat16)
    tasks, units_l, params = [], [[], []], bytearray()
    rr = 0
    n_ev = 1
    ops = [L.OP_ATTN_PARTIAL] + ([L.OP_ATTN_REDUCE] if reduce else [])
    for op in ops:
        for h in range(KVH):
            p = L.AttnParams()
            p.qkv, p.q_gamma, p.k_gamma = qkv.data_ptr(), g.data_ptr(), g.data_ptr()
            p.k_cache, p.v_cache = kc.data_ptr(), vc.data_ptr()
            p.rope_cos, p.rope_sin, p.positions = cos.data_ptr(), sin.data_ptr(), pos.data_ptr()
            p.partial, p.out = part.data_ptr(), out.data_ptr()
            p.M, p.ldqkv, p.q_heads, p.kv_heads, p.head_dim, p.group = B, (QH + 2 * KVH) * HD, QH, KVH, HD, G
            p.kv_head, p.split, p.n_splits, p.t_max = h, split, n_splits, t_max
            p.eps, p.scale, p.sub_splits = 1e-6, HD ** -0.5, sub
            items = B * n_splits if op == L.OP_ATTN_PARTIAL else B
            nu = min(units, items)
            t = L.Task(); t.op = op; t.level = L.LEVEL_CU; t.die = -1
            t.wait0 = t.wait1 = -1; t.signal = 0; t.n_items = items; t.n_units = nu
            t.sub_ctr = len(tasks) if nu > 1 else -1
            t.param_off = len(params); t.graph_index = -1
            params += bytes(p)
            ti = len(tasks)
            tasks.append(t)
            for u in range(nu):
                units_l[rr % 2].append((ti, u * items // nu, (u + 1) * items // nu))
                rr += 1
    flat = units_l[0] + units_l[1]
    t_arr = (L.Task * len(tasks))(*tasks)
    u_arr = (L.Unit * len(flat))(*[L.Unit(a, b, c, 0) for a, b, c in flat])
    b_arr = (C.c_int32 * 3)(0, len(units_l[0]), len(flat))
    r_arr = (C.c_int32 * 1)(len(tasks))
    pbuf = C.create_string_buffer(bytes(params), len(params))
    gd = L.GraphDesc(len(tasks), n_ev, len(flat), len(tasks), 2, L.SCHED_PER_DIE, W, len(params),
                     C.cast(t_arr, C.c_void_p), C.cast(r_arr, C.c_void_p),
                     C.cast(u_arr, C.c_void_p), C.cast(b_arr, C.c_void_p),
                     C.cast(pbuf, C.c_void_p))
    h = C.c_void_p()
    L.check(lib.mk_create(0, C.byref(gd), C.byref(topo), C.byref(h)))
    lib.mk_set_debug(h, debug)
    for _ in range(3):
        L.check(lib.mk_step(h, None))
        pos.fill_(T)
    L.check(lib.mk_sync(h))
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(steps):
        L.check(lib.mk_step(h, None))
    e1.record()
    torch.cuda.synchronize()
    L.check(lib.mk_sync(h))
    us = e0.elapsed_time(e1) / steps * 1e3
    if log:
        cap = 1 << 20
        lib.mk_log_enable(h, cap)
        pos.fill_(T)
        L.check(lib.mk_step(h, None))
        L.check(lib.mk_sync(h))
        buf = (L.LogRec * cap)()
        n = lib.mk_log_read(h, buf, cap)
        ph = {}
        ex = []
        for i in range(min(n, cap)):
            r = buf[i]
            if r.kind in (2, 3, 4):
                ph.setdefault(r.kind, []).append((r.t_end - r.t_start) / 1e3)
            if r.kind == 1:
                ex.append((r.t_start, r.t_end))
        t0 = min(a for a, _ in ex); t1 = max(b for _, b in ex)
        print("exec span us", (t1 - t0) / 1e3, "units", len(ex),
              "mean unit us", sum(b - a for a, b in ex) / len(ex) / 1e3)
        for k, v in sorted(ph.items()):
            print("phase", k, "n", len(v), "mean us", round(sum(v) / len(v), 3), "max", round(max(v), 3))
    lib.mk_destroy(h)
    return us


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "log":
        for B in (1, 64):
            print("B", B, run(B=B, units=19, sub=(2 if B == 1 else 1), log=True))
        sys.exit(0)
    res = []
    for B, units, sub, red in [(1, 19, 2, False), (1, 19, 1, False), (1, 19, 2, True), (8, 19, 1, False), (64, 19, 1, False)]:
        us = run(B=B, units=units, sub=sub, reduce=red)
        kv = B * 8 * 1024 * 128 * 2 * 2
        r = dict(B=B, units=units, sub=sub, reduce=red, us=round(us, 2), kv_gbs=round(kv / us / 1e3, 1))
        print(json.dumps(r), flush=True)
        res.append(r)
    # empty-graph floor: same launch, no work

