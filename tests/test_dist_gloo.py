"""Multi-process (gloo, world size 2) tests of the N>1 host logic.

* max-over-ranks timing used by bench.py;
* the TP partition plan: two ranks each compute their slice of a Qwen3
  decode step (fp32, CPU) with row-parallel allreduces, and the result equals
  the unsharded oracle step bit-for-bit up to fp32 reassociation.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tp_worker(rank, world, port, outq):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        from oracle.qwen3_fp32 import rms_norm, rotate_half
        from paper_2604_15379_b200 import dist as D
        from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights
        D.init("gloo")
        # max over ranks
        m = D.max_over_ranks(float(rank + 1))
        spec = Qwen3Spec(hidden=64, ffn=128, layers=2, q_heads=4, kv_heads=2,
                         head_dim=16, vocab=256)
        w = Qwen3Weights.random(spec, seed=3)
        plan = D.tp_plan(spec, world, rank)
        f32 = lambda t: t.float()  # noqa: E731
        B, hd = 2, spec.head_dim
        tok = torch.tensor([5, 77])
        x = f32(w.embed)[tok]
        pos = 0
        inv = 1.0 / (spec.rope_theta ** (torch.arange(0, hd, 2).float() / hd))
        fr = pos * inv
        emb = torch.cat((fr, fr))
        cos, sin = emb.cos(), emb.sin()
        for L in w.layers:
            h = rms_norm(x, f32(L["in_norm"]), spec.eps)
            qs = slice(plan.q_heads.start * hd, plan.q_heads.stop * hd)
            ks = slice(plan.kv_heads.start * hd, plan.kv_heads.stop * hd)
            q = (h @ f32(L["q"])[qs].T).view(B, -1, hd)
            k = (h @ f32(L["k"])[ks].T).view(B, -1, hd)
            v = (h @ f32(L["v"])[ks].T).view(B, -1, hd)
            q = rms_norm(q, f32(L["q_norm"]), spec.eps) * cos + rotate_half(rms_norm(q, f32(L["q_norm"]), spec.eps)) * sin
            k = rms_norm(k, f32(L["k_norm"]), spec.eps) * cos + rotate_half(rms_norm(k, f32(L["k_norm"]), spec.eps)) * sin
            # single cached token: softmax over one key = 1 -> output = v
            att = v.repeat_interleave(spec.group, dim=1)
            o_part = att.reshape(B, -1) @ f32(L["o"])[:, qs].T      # row-parallel
            dist.all_reduce(o_part)
            x = x + o_part
            h = rms_norm(x, f32(L["post_norm"]), spec.eps)
            fs = slice(plan.ffn.start, plan.ffn.stop)
            a = torch.nn.functional.silu(h @ f32(L["gate"])[fs].T) * (h @ f32(L["up"])[fs].T)
            d_part = a @ f32(L["down"])[:, fs].T                       # row-parallel
            dist.all_reduce(d_part)
            x = x + d_part
        h = rms_norm(x, f32(w.final_norm), spec.eps)
        vs = slice(plan.vocab.start, plan.vocab.stop)
        logits = h @ f32(w.lm_head)[vs].T
        val, idx = logits.max(-1)
        idx = idx + plan.vocab.start
        vals = [torch.zeros_like(val) for _ in range(world)]
        idxs = [torch.zeros_like(idx) for _ in range(world)]
        dist.all_gather(vals, val)
        dist.all_gather(idxs, idx)
        V = torch.stack(vals)
        I = torch.stack(idxs)
        best = V.argmax(0)                                  # lowest rank wins ties
        tokens = I.gather(0, best[None])[0]
        full = torch.cat([torch.zeros_like(logits)] * world, -1)
        parts = [torch.zeros_like(logits) for _ in range(world)]
        dist.all_gather(parts, logits)
        full = torch.cat(parts, -1)
        outq.put((rank, m, tokens.tolist(), full))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_tp2_decomposition_matches_unsharded_oracle():
    from oracle.qwen3_fp32 import Qwen3Fp32
    from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    assert res[0][1] == res[1][1] == 2.0
    spec = Qwen3Spec(hidden=64, ffn=128, layers=2, q_heads=4, kv_heads=2, head_dim=16, vocab=256)
    w = Qwen3Weights.random(spec, seed=3)
    o = Qwen3Fp32(w, t_max=4, batch=2)
    ref = o.step(torch.tensor([5, 77]))
    for r in res:
        assert torch.allclose(r[3], ref, atol=1e-5, rtol=1e-5)
        assert r[2] == ref.argmax(-1).tolist()


def test_tp_plan_partitions():
    from paper_2604_15379_b200.dist import allreduce_bytes_per_step, tp_plan
    from paper_2604_15379_b200.weights import Qwen3Spec
    spec = Qwen3Spec.qwen3_8b()
    for tp in (2, 4, 8):
        plans = [tp_plan(spec, tp, r) for r in range(tp)]
        assert sum(len(p.kv_heads) for p in plans) == 8
        assert sum(len(p.q_heads) for p in plans) == 32
        assert sum(len(p.ffn) for p in plans) == 12288
        assert sum(len(p.vocab) for p in plans) == 151936
        assert plans[-1].vocab.stop == 151936
    ab = allreduce_bytes_per_step(spec, 1)
    assert ab["calls"] == 72 and ab["bytes_per_call"] == 8192
    with pytest.raises(ValueError):
        tp_plan(spec, 3, 0)
