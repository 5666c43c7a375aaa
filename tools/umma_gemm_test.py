"""One tcgen05 GEMM die task per die vs torch: diagnose layout issues."""
import ctypes as C
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_15379_b200 import _lib as L
from paper_2604_15379_b200.runtime import probe, halves_topology
from paper_2604_15379_b200.weights import pack_umma


def run(N=512, K=128, M=16, mode="rand"):
    lib = L.load()
    topo = probe(0)
    if topo.num_dies != 2:
        topo = halves_topology(topo.num_sms)
    W = min(topo.sms_per_die[0], topo.sms_per_die[1]) - 1
    torch.manual_seed(0)
    if mode == "rand":
        w = torch.randn(N, K).to(torch.bfloat16)
        x = torch.randn(M, K).to(torch.bfloat16)
    elif mode == "eye":       # W = identity-ish: row r has a 1 at column r % K
        w = torch.zeros(N, K, dtype=torch.bfloat16)
        for r in range(N):
            w[r, r % K] = 1
        x = (torch.arange(M * K, dtype=torch.float32).view(M, K) % 251).to(torch.bfloat16)
    wp = pack_umma(w, 128, 64).cuda()
    xd = x.cuda()
    y = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    tasks, params = [], bytearray()
    n_loc = N // 2
    for d in range(2):
        p = L.GemmParams()
        p.w = wp.data_ptr() + d * n_loc * K * 2
        p.x, p.y = xd.data_ptr(), y.data_ptr()
        p.M, p.K, p.N = M, K, n_loc
        p.T_M, p.T_N, p.T_K = 16 if M <= 16 else M, 128, 64
        p.ldx, p.ldy, p.ldres = K, N, K
        p.y_col0 = d * n_loc
        p.epilogue = L.EPI_NONE
        p.traversal, p.distribution, p.xcd = L.TRAV_M_MAJOR, L.DIST_M_TILE, d
        p.tile_m = p.tile_n = -1
        p.body = L.BODY_UMMA
        p.y_cols = 1 << 30
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
    lib.mk_set_watchdog(h, 2.0)
    L.check(lib.mk_step(h, None))
    L.check(lib.mk_sync(h))
    lib.mk_destroy(h)
    ref = (x.float() @ w.float().T)
    got = y.float().cpu()
    return x, w, ref, got


if __name__ == "__main__":
    x, w, ref, got = run(mode="eye")
    print("eye: ref[0,:8]", ref[0, :8].tolist())
    print("eye: got[0,:8]", got[0, :8].tolist())
    print("eye: ref[1,:8]", ref[1, :8].tolist())
    print("eye: got[1,:8]", got[1, :8].tolist())
    print("eye: got[0,64:72]", got[0, 64:72].tolist(), "ref", ref[0, 64:72].tolist())
    # find for each output (b, r) which x column it matches
    xs = x.float()
    for b in (0, 1, 5):
        for r in (0, 1, 7, 8, 9, 31, 32, 64, 127, 128):
            v = got[b, r].item()
            cand = [(bb, k) for bb in range(x.shape[0]) for k in range(x.shape[1]) if xs[bb, k].item() == v]
            print(f"got[{b},{r}]={v} expected x[{b},{r % 128}]={xs[b, r % 128].item()} matches x at {cand[:4]}")
    x, w, ref, got = run(mode="rand")
    err = (got - ref).abs().max().item()
    print("rand: max abs err", err, "ref max", ref.abs().max().item())
