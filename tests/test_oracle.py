"""Pin the fp32 oracle (oracle/qwen3_fp32.py) against transformers' Qwen3ForCausalLM.

Fixtures: tests/golden/{toy,wide}_hf_logits.pt from oracle/gen_hf_golden.py.
"""

import os

import pytest
import torch

from oracle.qwen3_fp32 import Qwen3Fp32, greedy
from paper_2604_15379_b200.weights import (Qwen3Spec, Qwen3Weights, hash_uniform,
                                           pack_gate_up_fused, pack_tiles)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("name", ["toy_hf_logits.pt", "wide_hf_logits.pt"])
def test_oracle_matches_transformers(name):
    ref = torch.load(os.path.join(GOLD, name))
    spec = Qwen3Spec(**ref["spec"])
    w = Qwen3Weights.random(spec, seed=ref["seed"])
    tokens = ref["tokens"]
    B, T = tokens.shape
    o = Qwen3Fp32(w, t_max=T + 4, batch=B)
    for t in range(T):
        lg = o.step(tokens[:, t])
        want = ref["logits"][:, t]
        scale = want.abs().max().item()
        # fp32 vs fp32 with different summation order
        assert (lg - want).abs().max().item() <= 1e-4 * max(scale, 1.0), t
        assert torch.equal(greedy(lg), ref["greedy"][:, t])


def test_hash_init_is_device_independent_and_uniform():
    a = hash_uniform(1 << 16, seed=3, tid=11)
    b = hash_uniform(1 << 16, seed=3, tid=11)
    assert torch.equal(a, b)
    assert 0.0 <= a.min().item() and a.max().item() < 1.0
    assert abs(a.mean().item() - 0.5) < 0.01
    c = hash_uniform(1 << 16, seed=3, tid=12)
    assert not torch.equal(a, c)


def test_pack_tiles_layout():
    w = torch.arange(8 * 12, dtype=torch.float32).view(8, 12)
    p = pack_tiles(w, 4, 6)
    assert p.shape == (2, 2, 4, 6)
    assert torch.equal(p[1, 0], w[4:8, 0:6])
    assert torch.equal(p[0, 1], w[0:4, 6:12])


def test_pack_gate_up_fused_layout():
    g = torch.arange(8 * 4, dtype=torch.float32).view(8, 4)
    u = -g
    p = pack_gate_up_fused(g, u, dies=2, t_n=2, t_k=2)
    # die 1, tile 1, chunk 0: gate rows 6,7 then up rows 6,7, cols 0:2
    blk = p[1, 1, 0]
    assert torch.equal(blk[0], g[6:8, 0:2])
    assert torch.equal(blk[1], u[6:8, 0:2])


@torch.no_grad()
def test_bf16_restatement_matches_transformers_bf16():
    """Qwen3Fp32(dtype=bf16) -- the 36-layer GPU test's yardstick for the bf16
    format's own drift -- restates Qwen3ForCausalLM.to(bfloat16): decoded
    token by token on the toy model its logits are bit-identical to
    transformers' bf16 ones while the context is short (3 steps), and its
    drift from fp32 stays the size of transformers-bf16's afterwards (bf16
    matmul batching differs once the attention spans more keys)."""
    pytest.importorskip("transformers")
    from transformers import DynamicCache

    from oracle.gen_hf_golden import hf_model
    spec = Qwen3Spec.toy()
    w = Qwen3Weights.random(spec, seed=7)
    m = hf_model(w).to(torch.bfloat16)
    B, T = 2, 8
    tokens = torch.randint(0, spec.vocab, (B, T), generator=torch.Generator().manual_seed(5))
    o16 = Qwen3Fp32(w, t_max=T + 4, batch=B, dtype=torch.bfloat16)
    o32 = Qwen3Fp32(w, t_max=T + 4, batch=B)
    cache = DynamicCache()
    gaps16, gaps32 = [], []
    for t in range(T):
        out = m(input_ids=tokens[:, t:t + 1], past_key_values=cache, use_cache=True,
                position_ids=torch.full((B, 1), t, dtype=torch.long))
        cache = out.past_key_values
        hf16 = out.logits[:, 0].float()
        a, b = o16.step(tokens[:, t]), o32.step(tokens[:, t])
        assert a.dtype == torch.float32
        if t < 3:
            assert torch.equal(a, hf16), t
        scale = b.abs().max().item()
        gaps16.append((a - b).abs().max().item() / scale)
        gaps32.append((hf16 - b).abs().max().item() / scale)
    assert 0.5 * max(gaps32) <= max(gaps16) <= 2 * max(gaps32), (gaps16, gaps32)
