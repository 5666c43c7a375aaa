"""Golden logits from transformers' Qwen3ForCausalLM (test infrastructure).

Builds the toy Qwen3 (reference toy shapes, machine.py:189-196, + vocab 512)
and a 2-layer Qwen3-8B-width slice with the hash-initialised weights of
``paper_2604_15379_b200.weights``, runs transformers 5.5.0 ``Qwen3ForCausalLM``
in fp32 over a seeded prompt token by token (decode with a DynamicCache), and
saves prompt, per-step logits and greedy ids to ``tests/golden/*.pt``.
``tests/test_oracle.py`` pins ``oracle/qwen3_fp32.py`` against these.

    python oracle/gen_hf_golden.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights  # noqa: E402


def hf_model(w: Qwen3Weights, device="cpu"):
    from transformers import Qwen3Config, Qwen3ForCausalLM
    sp = w.spec
    cfg = Qwen3Config(vocab_size=sp.vocab, hidden_size=sp.hidden,
                      intermediate_size=sp.ffn, num_hidden_layers=sp.layers,
                      num_attention_heads=sp.q_heads,
                      num_key_value_heads=sp.kv_heads, head_dim=sp.head_dim,
                      rms_norm_eps=sp.eps, rope_theta=sp.rope_theta,
                      max_position_embeddings=4096, tie_word_embeddings=False,
                      attention_bias=False, hidden_act="silu")
    cfg._attn_implementation = "eager"
    with torch.device(device):
        m = Qwen3ForCausalLM(cfg).float().eval()
    sd = {"model.embed_tokens.weight": w.embed, "model.norm.weight": w.final_norm,
          "lm_head.weight": w.lm_head}
    for i, L in enumerate(w.layers):
        p = f"model.layers.{i}."
        sd.update({
            p + "self_attn.q_proj.weight": L["q"], p + "self_attn.k_proj.weight": L["k"],
            p + "self_attn.v_proj.weight": L["v"], p + "self_attn.o_proj.weight": L["o"],
            p + "self_attn.q_norm.weight": L["q_norm"],
            p + "self_attn.k_norm.weight": L["k_norm"],
            p + "mlp.gate_proj.weight": L["gate"], p + "mlp.up_proj.weight": L["up"],
            p + "mlp.down_proj.weight": L["down"],
            p + "input_layernorm.weight": L["in_norm"],
            p + "post_attention_layernorm.weight": L["post_norm"],
        })
    missing, unexpected = m.load_state_dict({k: v.float() for k, v in sd.items()},
                                            strict=False)
    assert not unexpected and all("rotary" in k for k in missing), (missing, unexpected)
    return m


@torch.no_grad()
def run(spec: Qwen3Spec, seed: int, batch: int, steps: int, name: str):
    from transformers import DynamicCache
    w = Qwen3Weights.random(spec, seed=seed)
    m = hf_model(w)
    g = torch.Generator().manual_seed(1234)
    tokens = torch.randint(0, spec.vocab, (batch, steps), generator=g)
    cache = DynamicCache()
    logits = []
    for t in range(steps):
        out = m(input_ids=tokens[:, t:t + 1], past_key_values=cache, use_cache=True,
                position_ids=torch.full((batch, 1), t, dtype=torch.long))
        cache = out.past_key_values
        logits.append(out.logits[:, 0].clone())
    logits = torch.stack(logits, 1)
    torch.save({"spec": spec.__dict__, "seed": seed, "tokens": tokens,
                "logits": logits, "greedy": logits.argmax(-1)},
               ROOT / "tests" / "golden" / name)
    print(name, tuple(logits.shape))


if __name__ == "__main__":
    run(Qwen3Spec.toy(), seed=7, batch=2, steps=12, name="toy_hf_logits.pt")
    run(Qwen3Spec(hidden=4096, ffn=12288, layers=1, q_heads=32, kv_heads=8,
                  head_dim=128, vocab=1024), seed=3, batch=1, steps=3,
        name="wide_hf_logits.pt")
