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


def _tp_lowering_worker(rank, world, port, outq):
    """Each gloo rank lowers ITS shard of the decode step with the product's
    tensor-parallel lowering (CPU buffers; nothing launched) and checks the
    descriptors, then the ranks cross-check each other through gloo."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        import ctypes
        from paper_2604_15379_b200 import _lib as L
        from paper_2604_15379_b200 import b200_from_probe, build_decoder_layer, model_preset
        from paper_2604_15379_b200 import dist as D
        from paper_2604_15379_b200.analytics import device_tiles
        from paper_2604_15379_b200.lowering import LoweringOptions, TPLayout, lower
        from paper_2604_15379_b200.runtime import _default_lm_tile, build_state
        from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights
        D.init("gloo")
        spec = Qwen3Spec.toy(layers=2)
        B = 2
        mach = b200_from_probe([74])                 # one rank = one die-sized SM set
        model = model_preset("toy")
        g = build_decoder_layer(model, mach, "chiplet", B,
                                tile_overrides=device_tiles(model, mach, "chiplet", B, tp=world),
                                layers=2)
        w = Qwen3Weights.random(spec, seed=5)
        ws = D.shard_weights(w, world, rank)
        sp = ws.spec
        lm = _default_lm_tile(sp, B)
        st = build_state(g, ws, 128, lm, sp.vocab // lm[1], device="cpu")
        layout = TPLayout(world, B, sp.hidden, 2)
        opts = LoweringOptions(sched_mode=L.SCHED_FLAT, workers=73, n_dies=1, lm_tile=lm,
                               tp_rank=rank, tp_world=world, tp_layout=layout)
        low = lower(g, sp, st, opts)
        names = low.task_names
        tasks = [low.tasks[i] for i in range(len(low.tasks))]
        ev = low.event_names

        def params(t, cls):
            return cls.from_buffer_copy(low.params[t.param_off:t.param_off + ctypes.sizeof(cls)])

        ars = [i for i, n in enumerate(names) if "allreduce" in n]
        assert len(ars) == 2 * 2                                     # o + down per layer
        for i in ars:
            t = tasks[i]
            assert t.op == L.OP_TP_ALLREDUCE and t.level == L.LEVEL_CU
            p = params(t, L.TPParams)
            point = 2 * t.layer + (0 if names[i].split(".")[1].startswith("o_") else 1)
            assert p.recv_off == layout.recv_off(point) and p.flag_off == layout.flag_off(point)
            # it waits on the partial GEMM's event and nothing else waits on that event
            gemm_ev = t.wait0
            assert ev[gemm_ev].endswith(("o_proj", "down"))
            waiters = [names[j] for j, u in enumerate(tasks) if u.wait0 == gemm_ev]
            assert waiters == [names[i]], waiters
            assert any(u.wait0 == t.signal for u in tasks), "someone consumes the sum"
        n_partial = 0
        for i, t in enumerate(tasks):
            if t.op != L.OP_GEMM:
                continue
            p = params(t, L.GemmParams)
            if p.epilogue == L.EPI_PARTIAL:
                n_partial += 1
                point = 2 * t.layer + (0 if ".o_proj." in names[i] else 1)
                assert (p.y or 0) == layout.slot_off(point, rank) and p.res is None
                assert p.K == (sp.q_heads * sp.head_dim if point % 2 == 0 else sp.ffn)
                assert p.N == sp.hidden
        assert n_partial == 2 * 2
        attn_items = {names[i]: t.n_items for i, t in enumerate(tasks) if t.op == L.OP_ATTN_PARTIAL}
        mine = {n for n, k in attn_items.items() if k > 0}
        assert mine == {f"L{l}.attn_partial.t{h}" for l in range(2)
                        for h in range(rank * sp.kv_heads, (rank + 1) * sp.kv_heads)}
        am = [t for t in tasks if t.op == L.OP_TP_ARGMAX]
        assert len(am) == 1 and params(am[0], L.TPParams).vocab0 == rank * sp.vocab
        # the ranks agree on the task / event order (flags and points line up)
        # and their shards tile the full weights exactly
        summ = dict(names=names, events=ev, layout=layout.nbytes,
                    q=ws.layers[0]["q"], o=ws.layers[0]["o"], down=ws.layers[1]["down"],
                    lm=ws.lm_head)
        allsum = [None] * world
        dist.all_gather_object(allsum, summ)
        assert all(a["names"] == names and a["events"] == ev and a["layout"] == layout.nbytes
                   for a in allsum)
        full = w.layers[0]
        ok = (torch.equal(torch.cat([a["q"] for a in allsum], 0), full["q"]) and
              torch.equal(torch.cat([a["o"] for a in allsum], 1), full["o"]) and
              torch.equal(torch.cat([a["down"] for a in allsum], 1), w.layers[1]["down"]) and
              torch.equal(torch.cat([a["lm"] for a in allsum], 0), w.lm_head))
        outq.put((rank, ok, len(tasks)))
    except Exception as e:  # surface the assertion to the parent
        import traceback
        outq.put((rank, traceback.format_exc(), 0))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_tp2_product_lowering_under_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_lowering_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] is True, r[1]
    assert res[0][2] == res[1][2]
