"""Tensor-parallel device path on ONE B200 (run on a B200: -m gpu).

The round's GPU boxes have one GPU, so a TP group of 2 ranks is emulated on
one device: each rank is its own Megakernel (its own shard of the weights,
descriptors, KV cache and exchange region) launched with 74 CTAs on its own
stream, so both persistent kernels run concurrently on disjoint SMs.  The
data path is the multi-GPU one: the row-parallel o_proj / down GEMMs push
their fp32 partials into BOTH ranks' exchange regions (MK_EPI_PARTIAL),
MK_OP_TP_ALLREDUCE exchanges release/acquire flags at system scope and sums
in rank order, MK_OP_TP_ARGMAX picks the global greedy token from the
vocab shards.  Only the peer pointers differ from a multi-GPU run (same
device memory here, NVLink peer / IPC mappings there: dist.connect_dist).

Checked against the unsharded fp32 oracle: the concatenated vocab-shard
logits within the north_star tolerance, greedy ids equal (near-ties
recorded), both ranks emitting the same tokens.
"""

import pytest
import torch

from oracle.qwen3_fp32 import Qwen3Fp32, margins

pytestmark = pytest.mark.gpu
RTOL = 2e-2


@pytest.fixture(scope="module")
def topo():
    from paper_2604_15379_b200.runtime import halves_topology, probe
    t = probe(0)
    return t if t.num_dies == 2 else halves_topology(t.num_sms)


def _group(spec, w, B, layers, topo, world=2, t_max=128):
    from dataclasses import replace
    from paper_2604_15379_b200 import b200_from_probe, build_decoder_layer, model_preset
    from paper_2604_15379_b200.analytics import device_tiles
    from paper_2604_15379_b200.dist import connect_local
    from paper_2604_15379_b200.runtime import Megakernel
    ctas = topo.num_sms // world
    mach = b200_from_probe([ctas])                  # one rank = one SM subset
    name = "toy" if spec.hidden == 64 else "qwen3-8b"
    model = replace(model_preset(name), num_layers=layers)
    g = build_decoder_layer(model, mach, "chiplet", B,
                            tile_overrides=device_tiles(model, mach, "chiplet", B, tp=world),
                            layers=layers)
    mks = [Megakernel(g, w, t_max=t_max, sched="flat", topo=topo, tp=(r, world),
                      ctas=ctas, cooperative=False, watchdog_s=10.0) for r in range(world)]
    connect_local(mks)
    return mks


def _run(mks, toks):
    streams = [torch.cuda.Stream() for _ in mks]
    for mk, st in zip(mks, streams):
        mk.set_tokens(toks)
        mk.launch(stream=st)
    for mk in mks:
        mk.sync()
    outs = [mk.state.out_tokens.cpu() for mk in mks]
    logits = torch.cat([mk.logits().float().cpu() for mk in mks], -1)
    return outs, logits


def _decode(mks, ref, B, steps, seed):
    gen = torch.Generator().manual_seed(seed)
    toks = torch.randint(0, ref.spec.vocab, (B,), generator=gen)
    worst, ties = 0.0, []
    for s in range(steps):
        outs, got = _run(mks, toks)
        want = ref.step(toks)
        assert all(torch.equal(o, outs[0]) for o in outs), "ranks disagree"
        diff = (got - want).abs()
        err = diff.max().item() / want.abs().max().item()
        worst = max(worst, err)
        assert err <= RTOL, (s, err)
        assert outs[0].tolist() == got.argmax(-1).tolist()      # global argmax of the shards
        marg = margins(want)
        for b in range(B):
            if outs[0][b].item() != want[b].argmax().item():
                assert marg[b].item() < 4 * diff.max().item(), (s, b)
                ties.append((s, b))
        toks = want.argmax(-1)
    return worst, ties


@pytest.mark.parametrize("B", [1, 4])
def test_tp2_toy_decode_on_one_gpu_matches_oracle(topo, B):
    from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights
    spec = Qwen3Spec.toy()
    w = Qwen3Weights.random(spec, seed=41)
    mks = _group(spec, w, B, 2, topo)
    ref = Qwen3Fp32(w, t_max=128, batch=B)
    for mk in mks:
        mk.set_positions([3 + 5 * b for b in range(B)])
    ref.pos[:] = torch.tensor([3 + 5 * b for b in range(B)])
    _decode(mks, ref, B, steps=4, seed=B)
    for mk in mks:
        mk.close()


def test_tp2_qwen3_8b_widths_on_one_gpu_matches_oracle(topo):
    """Qwen3-8B widths (d 4096, ffn 12288 -> 6144 per rank, 16 q / 4 kv heads
    per rank, vocab 151,936 -> 75,968 per rank), 2 layers, B=1."""
    from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights
    spec = Qwen3Spec.qwen3_8b(layers=2)
    w = Qwen3Weights.random(spec, seed=42, device="cuda")
    cpu = Qwen3Weights(w.spec, w.embed.float().cpu(), w.final_norm.float().cpu(),
                       w.lm_head.float().cpu(),
                       [{k: v.float().cpu() for k, v in L.items()} for L in w.layers])
    mks = _group(spec, w, 1, 2, topo)
    ref = Qwen3Fp32(cpu, t_max=128, batch=1)
    _decode(mks, ref, 1, steps=3, seed=7)
    for mk in mks:
        mk.close()


def _ipc_child(handle, nbytes, q):
    import ctypes as C
    import torch as T
    from paper_2604_15379_b200 import _lib as L
    lib = L.load()
    T.cuda.set_device(0)
    buf = (C.c_uint8 * 64).from_buffer_copy(handle)
    ptr = C.c_void_p()
    L.check(lib.mk_ipc_import(0, buf, C.byref(ptr)))
    # read the parent's pattern through the imported mapping, then write back
    n = nbytes // 4
    # wrap the raw device pointer with a torch tensor via __cuda_array_interface__
    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr.value, False),
                                    "version": 3}
    peer = T.as_tensor(_Arr(), device="cuda")
    ok = bool(T.equal(peer, T.arange(n, device="cuda", dtype=T.int32)))
    peer.mul_(2)
    T.cuda.synchronize()
    L.check(lib.mk_ipc_close(ptr))
    q.put(ok)


def test_exchange_region_ipc_between_processes():
    """dist.connect_dist's plumbing: an exchange region from mk_tp_alloc,
    exported with mk_ipc_export, opened by another process with
    mk_ipc_import -- both see the same device memory."""
    import ctypes as C
    import torch.multiprocessing as mp
    from paper_2604_15379_b200 import _lib as L
    lib = L.load()
    n = 1 << 16
    ptr = C.c_void_p()
    L.check(lib.mk_tp_alloc(0, 4 * n, C.byref(ptr)))

    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr.value, False),
                                    "version": 3}
    mine = torch.as_tensor(_Arr(), device="cuda")
    mine.copy_(torch.arange(n, device="cuda", dtype=torch.int32))
    torch.cuda.synchronize()
    h = (C.c_uint8 * 64)()
    L.check(lib.mk_ipc_export(ptr, h))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_ipc_child, args=(bytes(h), 4 * n, q))
    p.start()
    ok = q.get(timeout=120)
    p.join(timeout=60)
    assert ok and p.exitcode == 0
    assert torch.equal(mine, 2 * torch.arange(n, device="cuda", dtype=torch.int32))
    L.check(lib.mk_tp_free(ptr))
