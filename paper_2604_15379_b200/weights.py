"""Qwen3 weights: deterministic init and the packed HBM layouts the kernel streams.

Initialisation is a counter-based integer hash (identical bits on CPU and GPU,
no RNG state), so the fp32 CPU oracle and the device see the same bf16
weights without shipping checkpoints: ``w = bf16(a * (2u - 1))`` with
``u = hash(seed, tensor_id, index) / 2^24`` and ``a = std * sqrt(3)``
(uniform with the HF ``initializer_range`` std 0.02).

Canonical tensors follow the HF module layout
(``transformers/models/qwen3/modeling_qwen3.py``: ``nn.Linear`` weights are
``[out_features, in_features]``).  :func:`pack_tiles` rearranges a weight
matrix into the tile-major layout of the GEMM body: for tile ``n`` and
K-chunk ``c`` one contiguous ``[T_N, T_K]`` block, so a single TMA bulk copy
moves one shared-memory ring slot.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

_M32 = 0xFFFFFFFF


@dataclass(frozen=True)
class Qwen3Spec:
    """Qwen3 decoder shapes + numerics not carried by the reference ModelConfig."""

    hidden: int
    ffn: int
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int
    vocab: int
    eps: float = 1e-6
    rope_theta: float = 1e6

    @property
    def qkv_dim(self):
        return (self.q_heads + 2 * self.kv_heads) * self.head_dim

    @property
    def group(self):
        return self.q_heads // self.kv_heads

    @staticmethod
    def qwen3_8b(layers: int = 36, vocab: int = 151936):
        return Qwen3Spec(4096, 12288, layers, 32, 8, 128, vocab)

    @staticmethod
    def toy(layers: int = 2, vocab: int = 512):
        # the reference "toy" model (machine.py:189-196) + a small vocabulary
        return Qwen3Spec(64, 128, layers, 4, 2, 16, vocab)

    @staticmethod
    def from_model(model, vocab: int):
        return Qwen3Spec(model.hidden_dim, model.ffn_dim, model.num_layers,
                         model.q_heads, model.kv_heads, model.head_dim, vocab)


def hash_uniform(n: int, seed: int, tid: int, device="cpu",
                 chunk: int = 1 << 26) -> torch.Tensor:
    """Counter-based uniform [0,1) floats, bit-identical on every device."""
    out = torch.empty(n, dtype=torch.float32, device=device)
    salt = (seed * 0x27D4EB2D + tid * 0x165667B1 + 0x3C6EF372) & _M32
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        h = torch.arange(s, e, dtype=torch.int64, device=device)
        h = (h * 2654435761) & _M32
        h = h ^ salt
        for _ in range(3):
            h = (((h >> 16) ^ h) * 0x45D9F3B) & _M32
        h = (h >> 16) ^ h
        out[s:e] = (h >> 8).to(torch.float32) * (1.0 / (1 << 24))
    return out


def init_tensor(shape, seed, tid, std=None, center=0.0, half_width=None,
                device="cpu") -> torch.Tensor:
    n = math.prod(shape)
    u = hash_uniform(n, seed, tid, device)
    a = half_width if half_width is not None else std * math.sqrt(3.0)
    return (center + a * (2.0 * u - 1.0)).to(torch.bfloat16).view(*shape)


@dataclass
class Qwen3Weights:
    """Canonical (HF-layout) bf16 weights of one Qwen3 model."""

    spec: Qwen3Spec
    embed: torch.Tensor
    final_norm: torch.Tensor
    lm_head: torch.Tensor
    layers: list = field(default_factory=list)

    @staticmethod
    def random(spec: Qwen3Spec, seed: int = 0, device="cpu",
               std: float = 0.02, gamma_spread: float = 0.25,
               lm_std: float | None = None) -> "Qwen3Weights":
        d, f, hd = spec.hidden, spec.ffn, spec.head_dim
        tid = iter(range(1, 1 << 30))

        def lin(o, i, s=std):
            return init_tensor((o, i), seed, next(tid), std=s, device=device)

        def gam(n):
            return init_tensor((n,), seed, next(tid), center=1.0,
                               half_width=gamma_spread, device=device)

        embed = init_tensor((spec.vocab, d), seed, next(tid), std=std,
                            device=device)
        layers = []
        for _ in range(spec.layers):
            layers.append({
                "q": lin(spec.q_heads * hd, d),
                "k": lin(spec.kv_heads * hd, d),
                "v": lin(spec.kv_heads * hd, d),
                "o": lin(d, spec.q_heads * hd),
                "gate": lin(f, d),
                "up": lin(f, d),
                "down": lin(d, f),
                "q_norm": gam(hd),
                "k_norm": gam(hd),
                "in_norm": gam(d),
                "post_norm": gam(d),
            })
        final = gam(d)
        head = lin(spec.vocab, d, lm_std if lm_std is not None else std)
        return Qwen3Weights(spec, embed, final, head, layers)

    def to(self, device) -> "Qwen3Weights":
        mv = lambda t: t.to(device)  # noqa: E731
        return Qwen3Weights(self.spec, mv(self.embed), mv(self.final_norm),
                            mv(self.lm_head),
                            [{k: mv(v) for k, v in L.items()}
                             for L in self.layers])


def pack_tiles(w: torch.Tensor, t_n: int, t_k: int) -> torch.Tensor:
    """[N, K] -> tile-major [N/t_n, K/t_k, t_n, t_k] (contiguous)."""
    n, k = w.shape
    if n % t_n or k % t_k:
        raise ValueError(f"tile ({t_n},{t_k}) does not divide {tuple(w.shape)}")
    return (w.view(n // t_n, t_n, k // t_k, t_k).permute(0, 2, 1, 3)
            .contiguous())


def pack_gate_up_fused(gate: torch.Tensor, up: torch.Tensor, dies: int,
                       t_n: int, t_k: int) -> torch.Tensor:
    """Per die: tile n = [gate rows of tile n ; up rows of tile n] x K-chunk.

    Die ``x`` owns SiLU output columns ``[x*F/X, (x+1)*F/X)``, i.e. the
    reference slab ``[gate_local | up_local]`` (taskgraph.py:320-335), laid
    out so one 2*T_N-row block feeds one fused output tile.
    """
    f, k = gate.shape
    fl = f // dies
    if fl % t_n or k % t_k:
        raise ValueError("fused gate/up tile does not divide the slab")
    g = gate.view(dies, fl // t_n, t_n, k // t_k, t_k)
    u = up.view(dies, fl // t_n, t_n, k // t_k, t_k)
    both = torch.stack((g, u), dim=2)          # [X, nt, 2, t_n, kc, t_k]
    return both.permute(0, 1, 4, 2, 3, 5).contiguous()   # [X, nt, kc, 2, t_n, t_k]


def swizzle128(block: torch.Tensor) -> torch.Tensor:
    """Apply the 128-byte shared-memory swizzle to [..., rows, 64] bf16 blocks.

    K-major SWIZZLE_128B (the tcgen05 / TMA layout): a row is 128 bytes = eight
    16-byte chunks; inside every 8-row / 1024-byte atom, logical chunk c of
    row r is stored at chunk c ^ (r % 8).  Packing the weights this way in
    HBM lets a plain 1-D TMA bulk copy land a tile directly in the layout the
    UMMA shared-memory descriptor expects.
    """
    *lead, rows, cols = block.shape
    assert cols == 64
    v = block.reshape(*lead, rows, 8, 8)
    r = torch.arange(rows, device=block.device).view(rows, 1) % 8
    phys = torch.arange(8, device=block.device).view(1, 8)
    src = (phys ^ r)                                   # physical chunk <- logical chunk
    idx = src.view(*([1] * len(lead)), rows, 8, 1).expand(*lead, rows, 8, 8)
    return torch.gather(v, -2, idx).reshape(*lead, rows, cols)


def pack_umma(w: torch.Tensor, t_n: int = 128, t_k: int = 64) -> torch.Tensor:
    """[N, K] -> [N/t_n, K/t_k, t_n, t_k] tiles, each swizzled for tcgen05."""
    return swizzle128(pack_tiles(w, t_n, t_k)).contiguous()


def pack_gate_up_umma(gate: torch.Tensor, up: torch.Tensor, dies: int,
                      t_k: int = 64) -> torch.Tensor:
    """Fused gate/up die slabs for the tcgen05 body: a 128-row tile carries 64
    SiLU output columns, interleaved in 16-row groups [g 16q.., u 16q..] so
    that every 32-lane TMEM quadrant holds matching gate and up rows (the
    epilogue pairs them with one warp shuffle)."""
    f, k = gate.shape
    fl = f // dies
    if fl % 64 or k % t_k:
        raise ValueError("gate/up slab does not tile into 64-column UMMA tiles")
    g = gate.view(dies, fl // 64, 4, 16, k)
    u = up.view(dies, fl // 64, 4, 16, k)
    rows = torch.stack((g, u), dim=3).reshape(dies, fl // 64, 128, k)
    tiles = rows.view(dies, fl // 64, 128, k // t_k, t_k).permute(0, 1, 3, 2, 4)
    return swizzle128(tiles.contiguous()).contiguous()      # [X, nt, kc, 128, 64]


def pad_rows(w: torch.Tensor, multiple: int) -> torch.Tensor:
    n = w.shape[0]
    pad = (-n) % multiple
    if not pad:
        return w
    return torch.cat((w, torch.zeros(pad, *w.shape[1:], dtype=w.dtype, device=w.device)), 0)


def rope_tables(head_dim: int, theta: float, t_max: int):
    """cos/sin [t_max, head_dim/2] in fp32, as Qwen3RotaryEmbedding computes
    them (modeling_qwen3.py:112-150: inv_freq = 1/theta^(2i/d), freqs = p*inv)."""
    inv = 1.0 / (theta ** (torch.arange(0, head_dim, 2, dtype=torch.int64)
                           .to(torch.float32) / head_dim))
    pos = torch.arange(t_max, dtype=torch.float32)
    freqs = pos[:, None] * inv[None, :]
    return freqs.cos().contiguous(), freqs.sin().contiguous()
