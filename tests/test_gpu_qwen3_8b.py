"""GPU parity at the BENCHED configuration: Qwen3-8B widths (run on a B200: -m gpu).

Every test here builds the graph the bench builds -- d=4096, ffn=12288,
32 query / 8 kv heads (G=4), head_dim 128, vocab 151,936 -- and compares the
device decode step, through the C ABI, with the fp32 CPU oracle
(oracle/qwen3_fp32.py, pinned to transformers Qwen3ForCausalLM):

* 2-layer models at B in {1, 4, 16, 64}: the CUDA-core GEMV body (B=1), the
  tcgen05 body with 16-row (B=4, 16) and 64-row (B=64) activation tiles,
  die-task K-split pieces at d=4096 / ffn=12288, the padded 151,936 ->
  152,064-row LM head with masked tail columns, and the default tensor-core
  split-KV attention (one warp per item, separate ATTN_REDUCE) over a
  ~1024-token context: 16-17 64-token splits per row, per-row contexts that
  differ, so rows end in different splits at different offsets;
* the flat (die-unaware) scheduler on the same widths;
* the full 36-layer model at B=1 for 8 teacher-forced greedy steps.

The context is written once into both sides: canonical random K/V go to the
device cache through ``Megakernel.write_kv`` (which applies the tensor-core
path's chunk swizzle) and, upcast, into the oracle's fp32 cache.

Tolerances (north_star): logits within 2e-2 of the logit range (normwise:
max|dev - ref| / max|ref|; elementwise rtol is meaningless for logits near 0,
so the per-row relative L2 error is bounded too); greedy ids equal under
teacher forcing except at a recorded near-tie: a row whose top-1/top-2
oracle margin is below 4x the step's measured max absolute logit error.
Random-init weights make such rows common (151,936 nearly flat logits: oracle
margins of 1e-3..2e-2 against ~0.07 of bf16 error), so every step records
how many rows were ambiguous and which of them flipped; a flip on an
unambiguous row fails.
"""

import json
import os

import pytest
import torch

from oracle.qwen3_fp32 import Qwen3Fp32, margins

pytestmark = pytest.mark.gpu

RTOL = 2e-2          # north_star: bf16 device vs fp32 reference logits
# 36 layers: the bf16 format's own drift exceeds 2e-2.  transformers
# Qwen3ForCausalLM run in bf16 deviates from the same model in fp32 by
# 3.5-4.6 % normwise on these hash-initialised weights (the device: 3.1-5.2 %,
# same greedy ids) -- tools/precision_gap.py, profiles/r02/precision_gap_36.json.
# So the 36-layer test measures that drift itself, on the same context and
# tokens (the oracle restated with bf16 arithmetic, Qwen3Fp32(dtype=bf16)),
# and holds the device to DEEP_FACTOR x the bf16 model's own worst error
# (never tighter than RTOL).  At 2 layers both are ~1 % and 2e-2 applies.
DEEP_FACTOR = 1.5
ROW_L2 = 2e-2        # per-row ||dev - ref|| / ||ref|| (same rtol, L2 over the row)
CTX_LO, CTX_SPAN = 990, 90   # row b decodes at CTX_LO + (37 b) % CTX_SPAN
OUT = os.environ.get("MK_PARITY_OUT", "gpurun_out/parity")


@pytest.fixture(scope="module")
def topo():
    from paper_2604_15379_b200.runtime import halves_topology, probe
    t = probe(0)
    return t if t.num_dies == 2 else halves_topology(t.num_sms)


@pytest.fixture(scope="module")
def machine(topo):
    from paper_2604_15379_b200 import b200_from_probe
    return b200_from_probe([topo.sms_per_die[i] for i in range(topo.num_dies)])


def _weights(layers, seed):
    from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights
    w = Qwen3Weights.random(Qwen3Spec.qwen3_8b(layers=layers), seed=seed, device="cuda")
    cpu = Qwen3Weights(w.spec, w.embed.float().cpu(), w.final_norm.float().cpu(),
                       w.lm_head.float().cpu(),
                       [{k: v.float().cpu() for k, v in L.items()} for L in w.layers])
    return w, cpu


@pytest.fixture(scope="module")
def w2():
    return _weights(2, seed=21)


def _graph(machine, mode, B, layers):
    from dataclasses import replace
    from paper_2604_15379_b200 import build_decoder_layer, model_preset
    from paper_2604_15379_b200.analytics import device_tiles
    model = replace(model_preset("qwen3-8b"), num_layers=layers)
    return build_decoder_layer(model, machine, mode, B,
                               tile_overrides=device_tiles(model, machine, mode, B),
                               layers=layers)


def _context(mk, ref, B, seed, ref16=None):
    """Random canonical K/V for tokens [0, max pos) into both caches."""
    from paper_2604_15379_b200.weights import hash_uniform
    sp = mk.spec
    pos = torch.tensor([CTX_LO + (37 * b) % CTX_SPAN for b in range(B)])
    n = int(pos.max())
    for li in range(len(mk.state.k_cache)):
        kv = []
        for j in range(2):
            u = hash_uniform(B * sp.kv_heads * n * sp.head_dim, seed, 2 * li + j, device="cuda")
            kv.append(((u * 2 - 1) * 1.7).to(torch.bfloat16).view(B, sp.kv_heads, n, sp.head_dim))
        mk.write_kv(li, kv[0], kv[1], n)
        ref.load_kv(li, kv[0].float().cpu(), kv[1].float().cpu(), n)
        if ref16 is not None:
            ref16.load_kv(li, kv[0], kv[1], n)
    mk.set_positions(pos)
    ref.pos[:] = pos
    if ref16 is not None:
        ref16.pos[:] = pos
    return pos


def decode_vs_oracle(mk, ref, B, steps, seed, tag, rtol=RTOL, ref16=None):
    """Teacher-forced decode; returns a per-step report (written to OUT).

    With ``ref16`` (the bf16-arithmetic restatement on the same context) the
    tolerance is DEEP_FACTOR x its worst error against the fp32 oracle."""
    gen = torch.Generator().manual_seed(seed)
    toks = torch.randint(0, mk.spec.vocab, (B,), generator=gen)
    report, ties = [], []
    for s in range(steps):
        out = mk.step(toks).cpu()
        want = ref.step(toks)
        got = mk.logits().float().cpu()
        diff = (got - want).abs()
        scale = want.abs().max().item()
        err = diff.max().item() / scale
        row_l2 = ((got - want).norm(dim=-1) / want.norm(dim=-1)).max().item()
        extra = {}
        if ref16 is not None:
            w16 = ref16.step(toks)
            extra = dict(bf16_normwise_err=(w16 - want).abs().max().item() / scale,
                         bf16_row_l2_err=((w16 - want).norm(dim=-1) / want.norm(dim=-1)).max().item(),
                         bf16_ids=w16.argmax(-1).tolist())
        marg = margins(want)
        dev_ids, ref_ids = out.tolist(), want.argmax(-1).tolist()
        # the device argmax is the argmax of the device's own logits (lowest
        # index wins ties, as torch.argmax)
        assert dev_ids == got.argmax(-1).tolist(), (tag, s)
        tol = 4 * diff.max().item()
        ambiguous = [b for b in range(B) if marg[b].item() < tol]
        step_ties = []
        for b in range(B):
            if dev_ids[b] != ref_ids[b]:
                rec = dict(step=s, row=b, margin=marg[b].item(), tie_tol=tol,
                           dev=dev_ids[b], ref=ref_ids[b])
                assert rec["margin"] < tol, ("greedy id mismatch outside a near-tie", tag, rec)
                step_ties.append(rec)
        ties += step_ties
        report.append(dict(step=s, normwise_err=err, row_l2_err=row_l2,
                           min_margin=marg.min().item(), tie_tol=tol,
                           n_ambiguous=len(ambiguous), n_flipped=len(step_ties), **extra))
        if ref16 is None:
            assert err <= rtol, (tag, s, err)
            assert row_l2 <= max(ROW_L2, rtol), (tag, s, row_l2)
        toks = want.argmax(-1)
    summary = {}
    if ref16 is not None:
        tol_n = max(rtol, DEEP_FACTOR * max(r["bf16_normwise_err"] for r in report))
        tol_r = max(ROW_L2, DEEP_FACTOR * max(r["bf16_row_l2_err"] for r in report))
        summary = dict(deep_factor=DEEP_FACTOR, normwise_tol=tol_n, row_l2_tol=tol_r)
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"{tag}.json"), "w") as f:
        json.dump(dict(tag=tag, batch=B, steps=report, ties=ties, **summary,
                       positions_end=mk.positions().tolist()), f, indent=1)
    if ref16 is not None:
        for r in report:
            assert r["normwise_err"] <= summary["normwise_tol"], (tag, r)
            assert r["row_l2_err"] <= summary["row_l2_tol"], (tag, r)
    return report, ties


@pytest.mark.parametrize("B", [1, 4, 16, 64])
def test_qwen3_8b_widths_decode_matches_oracle(topo, machine, w2, B):
    import ctypes
    from paper_2604_15379_b200 import _lib as L
    from paper_2604_15379_b200.runtime import Megakernel
    w, cpu = w2
    g = _graph(machine, "chiplet", B, 2)
    mk = Megakernel(g, w, t_max=1152, topo=topo, watchdog_s=10.0)
    low = mk.lowered
    bodies, ksplit, attn = set(), 0, set()
    for i in range(len(low.tasks)):
        t = low.tasks[i]
        if t.op == L.OP_GEMM:
            p = L.GemmParams.from_buffer_copy(
                low.params[t.param_off:t.param_off + ctypes.sizeof(L.GemmParams)])
            bodies.add(p.body)
            ksplit += p.ksplit
        if t.op == L.OP_ATTN_PARTIAL:
            p = L.AttnParams.from_buffer_copy(
                low.params[t.param_off:t.param_off + ctypes.sizeof(L.AttnParams)])
            attn.add((p.mma, p.sub_splits, p.fuse_reduce, p.group, p.n_splits))
    # the configuration the bench runs at this batch
    from paper_2604_15379_b200.analytics import UMMA_MIN_BATCH
    assert bodies == ({L.BODY_GEMV} if B < UMMA_MIN_BATCH else {L.BODY_UMMA})
    assert attn == {(1, 1, 0, 4, 18)} and mk.kv_swizzled
    if B >= UMMA_MIN_BATCH:
        assert mk.state.vocab_pad == 152064 and ksplit > 0
    ref = Qwen3Fp32(cpu, t_max=1152, batch=B)
    _context(mk, ref, B, seed=40 + B)
    decode_vs_oracle(mk, ref, B, steps=3, seed=B, tag=f"qwen3_8b_2l_b{B}")
    mk.close()


def test_qwen3_8b_widths_flat_scheduler_matches_oracle(topo, machine, w2):
    """The die-unaware baseline (standard graph, one scheduler) at B=16."""
    from paper_2604_15379_b200.runtime import Megakernel
    w, cpu = w2
    B = 16
    g = _graph(machine, "standard", B, 2)
    mk = Megakernel(g, w, t_max=1152, topo=topo, sched="flat", watchdog_s=10.0)
    ref = Qwen3Fp32(cpu, t_max=1152, batch=B)
    _context(mk, ref, B, seed=77)
    decode_vs_oracle(mk, ref, B, steps=2, seed=5, tag="qwen3_8b_2l_b16_flat")
    mk.close()


def test_kv_write_read_roundtrip(topo, machine, w2):
    """write_kv / read_kv are inverse, and the swizzle is a per-row chunk
    permutation."""
    from paper_2604_15379_b200.runtime import Megakernel
    w, _ = w2
    g = _graph(machine, "chiplet", 2, 2)
    mk = Megakernel(g, w, t_max=128, topo=topo)
    k = torch.randn(2, 8, 100, 128, device="cuda").to(torch.bfloat16)
    v = torch.randn(2, 8, 100, 128, device="cuda").to(torch.bfloat16)
    mk.write_kv(1, k, v, 100)
    k2, v2 = mk.read_kv(1, 100)
    assert torch.equal(k2, k) and torch.equal(v2, v)
    raw = mk.state.k_cache[1][:, :, :100]
    # the stored row holds the same 16-byte chunks, permuted
    def chunks(x):   # per-row multiset of 16-byte chunks (as exact int64 keys)
        c = x.contiguous().view(torch.int16).to(torch.int64).view(2, 8, 100, 16, 8) & 0xFFFF
        key = (c[..., 0] << 48) | (c[..., 1] << 32) | (c[..., 2] << 16) | c[..., 3]
        key = key * 1000003 + ((c[..., 4] << 48) | (c[..., 5] << 32) | (c[..., 6] << 16) | c[..., 7])
        return key.sort(-1).values
    assert torch.equal(chunks(raw), chunks(k))
    assert not torch.equal(raw, k)
    mk.close()


def test_position_past_cache_is_refused(topo, machine, w2):
    """a row at t_max must not index past the cache -- the host
    refuses the launch, and a device-side overrun (positions written
    behind the wrapper's back) comes back as MK_ERR_CONFIG from mk_sync."""
    from paper_2604_15379_b200 import _lib as L
    from paper_2604_15379_b200.runtime import Megakernel
    w, _ = w2
    g = _graph(machine, "chiplet", 1, 2)
    mk = Megakernel(g, w, t_max=128, topo=topo)
    with pytest.raises(ValueError):
        mk.set_positions([128])
    mk.set_positions([127])
    mk.step([5])                       # appends at 127: the last row
    with pytest.raises(L.MkError):
        mk.launch()                    # would append at 128
    mk.state.positions.fill_(130)      # bypass the host check
    L.check(mk.lib.mk_step(mk.h, None))
    with pytest.raises(L.MkError) as ei:
        mk.sync()
    assert ei.value.code == L.MK_ERR_CONFIG and b"outside the KV cache" in mk.lib.mk_last_error()
    mk.set_positions([3])              # the handle recovers
    mk.step([7])
    mk.close()


def test_qwen3_8b_36_layers_greedy_and_sync_accounting(topo, machine):
    """The benched model itself (36 layers, B=1): 8 teacher-forced greedy
    steps at a ~1024-token context vs the fp32 oracle, then the sync
    accounting of one step (fan-out off, as the reference dispatches whole
    tasks) == the reference simulator's at the probed W
    (oracle/sched_accounting.py, pinned to ref simulate() for W in 64..77 by
    tests/golden/sim_counters_w.json)."""
    from oracle.sched_accounting import expected_counters
    from paper_2604_15379_b200.runtime import Megakernel
    w, cpu = _weights(36, seed=0)
    g = _graph(machine, "chiplet", 1, 36)
    mk = Megakernel(g, w, t_max=1152, topo=topo, watchdog_s=10.0)
    ref = Qwen3Fp32(cpu, t_max=1152, batch=1)
    ref16 = Qwen3Fp32(w, t_max=1152, batch=1, dtype=torch.bfloat16, device="cuda")
    _context(mk, ref, 1, seed=3, ref16=ref16)
    del cpu
    decode_vs_oracle(mk, ref, 1, steps=8, seed=9, tag="qwen3_8b_36l_b1", ref16=ref16)
    mk.close()
    del ref, ref16
    mk = Megakernel(g, w, t_max=64, topo=topo, fanout=False, watchdog_s=10.0)
    mk.set_positions([10])
    mk.reset_counters()
    mk.step([3])
    c = mk.counters()
    mk.close()
    X, W = machine.num_xcds, machine.workers_per_xcd
    exp = expected_counters(g, W)
    # appended head (final_norm, lm_head per die, argmax), absent from the
    # reference graph: 2 + X dispatches, X fences, X*W local atomics,
    # 2 + X global atomics
    got = {"dispatches": c["dispatches"] - (2 + X), "fences": c["fences"] - X,
           "local_atomics": c["local_atomics"] - X * W,
           "global_atomics": c["global_atomics"] - (2 + X)}
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "sync_accounting_36l.json"), "w") as f:
        json.dump(dict(workers_per_die=W, dies=X, expected=exp, device=got), f, indent=1)
    for k in ("dispatches", "fences", "local_atomics", "global_atomics"):
        assert got[k] == exp[k], (k, got[k], exp[k])
