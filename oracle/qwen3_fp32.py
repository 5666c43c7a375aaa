"""fp32 CPU restatement of one Qwen3 decode step -- TEST INFRASTRUCTURE ONLY.

The reference (chipletsim) carries no numerics, so
logits / greedy token ids are pinned by a third-party restatement:
transformers 5.5.0 ``Qwen3ForCausalLM`` (not vendored in the reference).
This module re-states its decode math in plain fp32 torch, line by line:

* RMSNorm: fp32 statistics, ``x * rsqrt(mean(x^2) + eps)``, then ``* gamma``
  (modeling_qwen3.py:50-64);
* q/k projections -> per-head q_norm / k_norm over head_dim
  (modeling_qwen3.py:263-264);
* RoPE ``x*cos + rotate_half(x)*sin`` with ``inv_freq = 1/theta^(2i/d)``
  (modeling_qwen3.py:112-181);
* GQA attention, softmax in fp32, scaling ``head_dim**-0.5``
  (modeling_qwen3.py:196-219, 235);
* residual adds and the SiLU MLP (modeling_qwen3.py:70-82, 315-333);
* final norm + LM head (modeling_qwen3.py:442-505), argmax with the lowest
  index winning ties (``torch.argmax``).

The weights are the same bf16 tensors the device uses, upcast to fp32; the
restatement is cross-checked against ``Qwen3ForCausalLM`` itself by
``tests/test_oracle.py`` (fixture ``tests/golden/toy_hf_logits.pt`` made by
``oracle/gen_hf_golden.py``).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg may import this module.
"""

from __future__ import annotations

import torch


def rms_norm(x: torch.Tensor, g: torch.Tensor, eps: float) -> torch.Tensor:
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g


def rotate_half(x: torch.Tensor) -> torch.Tensor:
    h = x.shape[-1] // 2
    return torch.cat((-x[..., h:], x[..., :h]), dim=-1)


class Qwen3Fp32:
    """Sequential decode with an fp32 KV cache, batch rows independent.

    ``dtype=torch.bfloat16`` (on any ``device``) instead restates the same
    model executed the way ``Qwen3ForCausalLM.to(torch.bfloat16)`` executes
    it: bf16 weights, activations and KV cache, every op rounding its output
    to bf16, RMSNorm statistics and the softmax in fp32 then cast back
    (modeling_qwen3.py:50-64, 196-219).  It is not the oracle: the GPU
    parity test uses it to measure the bf16 format's own drift from fp32 at
    36 layers, the yardstick the device's deviation is held to."""

    def __init__(self, weights, t_max: int, batch: int, dtype=torch.float32, device="cpu"):
        sp = weights.spec
        self.spec = sp
        self.dt = dtype
        f32 = lambda t: t.detach().to(device, dtype)  # noqa: E731
        self.embed = f32(weights.embed)
        self.final_norm = f32(weights.final_norm)
        self.lm_head = f32(weights.lm_head)
        self.layers = [{k: f32(v) for k, v in L.items()} for L in weights.layers]
        self.t_max = t_max
        self.batch = batch
        hd = sp.head_dim
        inv = 1.0 / (sp.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.int64)
                                       .to(torch.float32) / hd))
        pos = torch.arange(t_max, dtype=torch.float32)
        freqs = pos[:, None] * inv[None, :]
        emb = torch.cat((freqs, freqs), dim=-1)
        self.cos, self.sin = emb.cos().to(device, dtype), emb.sin().to(device, dtype)
        self.k = [torch.zeros(batch, sp.kv_heads, t_max, hd, device=device, dtype=dtype)
                  for _ in self.layers]
        self.v = [torch.zeros(batch, sp.kv_heads, t_max, hd, device=device, dtype=dtype)
                  for _ in self.layers]
        self.pos = torch.zeros(batch, dtype=torch.int64)

    def load_kv(self, layer: int, k: torch.Tensor, v: torch.Tensor, n: int):
        """Seed the cache with ``n`` tokens (fp32 copies of device bf16 KV)."""
        self.k[layer][:, :, :n] = k[:, :, :n].to(self.k[layer])
        self.v[layer][:, :, :n] = v[:, :, :n].to(self.v[layer])

    @torch.no_grad()
    def step(self, tokens: torch.Tensor, layers: int | None = None) -> torch.Tensor:
        """Decode one token per row at ``self.pos``; returns fp32 logits [B, V]."""
        sp = self.spec
        B, hd, G = tokens.shape[0], sp.head_dim, sp.group
        rms_norm = self._norm
        x = self.embed[tokens.long().to(self.embed.device)]  # [B, d]
        n_layers = len(self.layers) if layers is None else layers
        for li in range(n_layers):
            L = self.layers[li]
            h = rms_norm(x, L["in_norm"], sp.eps)
            q = (h @ L["q"].T).view(B, sp.q_heads, hd)
            k = (h @ L["k"].T).view(B, sp.kv_heads, hd)
            v = (h @ L["v"].T).view(B, sp.kv_heads, hd)
            q = rms_norm(q, L["q_norm"], sp.eps)
            k = rms_norm(k, L["k_norm"], sp.eps)
            out = torch.empty(B, sp.q_heads, hd, device=x.device, dtype=x.dtype)
            for b in range(B):
                p = int(self.pos[b])
                c, s = self.cos[p], self.sin[p]
                qb = q[b] * c + rotate_half(q[b]) * s
                kb = k[b] * c + rotate_half(k[b]) * s
                self.k[li][b, :, p] = kb
                self.v[li][b, :, p] = v[b]
                keys = self.k[li][b, :, :p + 1]             # [kvh, T, hd]
                vals = self.v[li][b, :, :p + 1]
                keys = keys.repeat_interleave(G, dim=0)      # repeat_kv
                vals = vals.repeat_interleave(G, dim=0)
                att = (qb[:, None, :] @ keys.transpose(1, 2)) * hd ** -0.5
                att = torch.softmax(att.float(), dim=-1).to(att.dtype)
                out[b] = (att @ vals)[:, 0, :]
            x = x + out.reshape(B, -1) @ L["o"].T
            h = rms_norm(x, L["post_norm"], sp.eps)
            g = h @ L["gate"].T
            u = h @ L["up"].T
            x = x + (torch.nn.functional.silu(g) * u) @ L["down"].T
        self.pos += 1
        h = rms_norm(x, self.final_norm, sp.eps)
        return (h @ self.lm_head.T).float().cpu()

    def _norm(self, x: torch.Tensor, g: torch.Tensor, eps: float) -> torch.Tensor:
        if self.dt == torch.float32:
            return rms_norm(x, g, eps)
        # Qwen3RMSNorm under bf16: fp32 statistics, cast, then gamma in bf16
        xf = x.float()
        return g * (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype)


def greedy(logits: torch.Tensor) -> torch.Tensor:
    return torch.argmax(logits, dim=-1)


def margins(logits: torch.Tensor) -> torch.Tensor:
    """top-1 minus top-2 logit per row (near-tie detector)."""
    top = torch.topk(logits, 2, dim=-1).values
    return top[:, 0] - top[:, 1]
