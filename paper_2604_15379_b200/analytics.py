"""Closed-form locality / roofline models and the decode-step byte budget.

The first three functions restate the reference's pure formulas
(``/root/reference/pkg/src/chipletsim/analytics.py:27-49``) and are used as
the *predicted* column next to measured L2 hit rates.  :func:`fit_tiles`
follows ``scenario.py:83-106``.  :func:`decode_step_bytes` is the algorithmic
HBM byte count of one decode step that ``bench.py`` divides by the measured
step time.
"""

from __future__ import annotations

import os

from .machine import MachineConfig, ModelConfig
from .taskgraph import LINEAR_OPS, STANDARD_TILE_PROFILE, OpKind


class AnalyticsError(ValueError):
    pass


def weight_hit_model(workers: int, batch: int, t_m: int) -> float:
    """(R-1)/R with R = min(W, ceil(B/T_M)) (ref analytics.py:27-33)."""
    if min(workers, batch, t_m) < 1:
        raise AnalyticsError("workers, batch, and t_m must be positive")
    r = min(workers, -(-batch // t_m))
    return 1.0 - 1.0 / r


def effective_ai(batch: int, l2_hit_rate: float) -> float:
    """B / (1 - h) (ref analytics.py:36-42)."""
    if batch < 1:
        raise AnalyticsError("batch must be positive")
    if not (0.0 <= l2_hit_rate < 1.0):
        raise AnalyticsError("l2_hit_rate must lie in [0, 1)")
    return batch / (1.0 - l2_hit_rate)


def roofline(ai: float, machine: MachineConfig) -> float:
    """min(peak, bw * ai) (ref analytics.py:45-49)."""
    if ai < 0:
        raise AnalyticsError("arithmetic intensity must be nonnegative")
    return min(machine.peak_flops, machine.hbm_bandwidth_bytes_per_s * ai)


def linear_gemm_dims(op: OpKind, model: ModelConfig) -> tuple:
    """(K, N) of a linear op (ref analytics.py:71-83)."""
    table = {
        OpKind.QKV_PROJ: (model.hidden_dim, model.qkv_dim),
        OpKind.O_PROJ_RESIDUAL: (model.hidden_dim, model.hidden_dim),
        OpKind.GATE_UP_SILU: (model.hidden_dim, model.gate_up_dim),
        OpKind.DOWN_PROJ_RESIDUAL: (model.ffn_dim, model.hidden_dim),
    }
    if op not in table:
        raise AnalyticsError(f"{op.value} is not a linear op")
    return table[op]


def shard_gemm_dims(op: OpKind, model: ModelConfig, tp: int = 1) -> tuple:
    """(K, N) of one tensor-parallel rank's shard of a linear op: QKV and
    gate/up column-parallel (N / tp), O and down row-parallel (K / tp)."""
    k, n = linear_gemm_dims(op, model)
    if op in (OpKind.QKV_PROJ, OpKind.GATE_UP_SILU):
        return k, n // tp
    return k // tp, n


def fit_tiles(model: ModelConfig, machine: MachineConfig, graph_mode: str,
              base: dict | None = None) -> dict:
    """Halve T_N / T_K until they divide the model's GEMMs (ref scenario.py:83-106).

    ``base`` optionally replaces the starting tiles (the reference starts
    from the standard profile or 16x64x256).
    """
    out = {}
    for op in LINEAR_OPS:
        k, n = linear_gemm_dims(op, model)
        width = n if graph_mode == "standard" else n // machine.num_xcds
        if op is OpKind.GATE_UP_SILU and graph_mode == "chiplet":
            width //= 2
        if base is not None:
            t_m, t_n, t_k = base[op]
        elif graph_mode == "standard":
            t_m, t_n, t_k = STANDARD_TILE_PROFILE[op]
        else:
            t_m, t_n, t_k = (16, 64, 256)
        while width % t_n:
            t_n //= 2
        while k % t_k:
            t_k //= 2
        out[op] = (t_m, t_n, t_k)
    out["silu_chunk"] = min(STANDARD_TILE_PROFILE["silu_chunk"], model.ffn_dim)
    return out


# batch rows from which the tcgen05 body is used (MK_UMMA_MIN_BATCH overrides)
UMMA_MIN_BATCH = int(os.environ.get("MK_UMMA_MIN_BATCH", "3"))
UMMA_MAX_TM = 64         # batch rows per tcgen05 m-tile (UMMA N, TMEM columns)


def default_t_m(batch: int) -> int:
    """Batch rows per m-tile: 16 for the CUDA-core GEMV (register budget),
    the whole batch (up to 64, padded to 16) for the tcgen05 body so every
    weight tile is streamed from HBM once per step."""
    if batch >= UMMA_MIN_BATCH:
        return min(UMMA_MAX_TM, -(-batch // 16) * 16)
    return 16


def umma_tiles(model: ModelConfig, machine: MachineConfig, graph_mode: str,
               t_m: int = 16) -> dict:
    """Tiles of the tcgen05 body: 128 weight rows (UMMA M) x 64-wide K chunks
    (one 128B-swizzled 16 KiB ring slot); the fused gate/up die task carries
    64 SiLU columns (64 gate + 64 up rows) per tile."""
    out = {}
    for op in LINEAR_OPS:
        fused = op is OpKind.GATE_UP_SILU and graph_mode == "chiplet"
        out[op] = (t_m, 64 if fused else 128, 64)
    out["silu_chunk"] = min(STANDARD_TILE_PROFILE["silu_chunk"], model.ffn_dim)
    return out


def device_tiles(model: ModelConfig, machine: MachineConfig, graph_mode: str,
                 batch: int = 1, t_m: int | None = None, umma: bool | None = None,
                 tp: int = 1) -> dict:
    """Tile overrides for the device GEMM bodies: the tcgen05 body from
    UMMA_MIN_BATCH rows per m-tile on (when every per-task width divides its
    128-row tiles), the CUDA-core warp-row GEMV below (see gemv_tiles).
    ``tp``: tiles of one tensor-parallel rank's shard (shard_gemm_dims)."""
    if t_m is None:
        t_m = default_t_m(batch)
    use = umma if umma is not None else min(batch, t_m) >= UMMA_MIN_BATCH
    if use:
        tiles = umma_tiles(model, machine, graph_mode, t_m)
        ok = True
        for op in LINEAR_OPS:
            k, n = shard_gemm_dims(op, model, tp)
            width = n if graph_mode == "standard" else n // machine.num_xcds
            rows = 128 if not (op is OpKind.GATE_UP_SILU and graph_mode == "chiplet") else 128
            if op is OpKind.GATE_UP_SILU and graph_mode == "chiplet":
                width //= 2
                rows = 64
            ok = ok and width % rows == 0 and k % 64 == 0
        if ok:
            return tiles
    return gemv_tiles(model, machine, graph_mode, batch, min(t_m, 16), tp)


def gemv_tiles(model: ModelConfig, machine: MachineConfig, graph_mode: str,
               batch: int = 1, t_m: int = 16, tp: int = 1) -> dict:
    """B200 tile overrides for the warp-row GEMM body (csrc gemm_tile).

    One shared-memory ring slot holds ``R x T_K`` bf16 (16 KiB) with
    ``R = T_N`` rows (``2*T_N`` for the fused gate/up die task); each of the 8
    consumer warps owns ``R/8`` rows.  More rows per warp amortise the
    activation reads over more weights, so R grows with the batch rows per
    m-tile: 8 rows for one row, 16 for up to 4, 32 beyond.  ``T_K`` is
    ``8192 / R`` (or K itself when K < 256).  Passing the result as
    ``tile_overrides`` to both builders keeps graph parity.
    """
    rows = min(batch, t_m)
    r_plain = 16 if rows <= 4 else 32
    r_fused = 16 if rows <= 4 else 32
    if os.environ.get("MK_GEMV_ROWS"):     # A/B knob: weight rows per ring slot
        r_plain = r_fused = int(os.environ["MK_GEMV_ROWS"])
    out = {}
    for op in LINEAR_OPS:
        k, n = shard_gemm_dims(op, model, tp)
        fused = op is OpKind.GATE_UP_SILU and graph_mode == "chiplet"
        width = n if graph_mode == "standard" else n // machine.num_xcds
        if fused:
            width //= 2
        r = r_fused if fused else r_plain
        tn = r // 2 if fused else r
        while width % tn and tn > (4 if fused else 8):
            tn //= 2
        r = 2 * tn if fused else tn
        tk = min(8192 // r, k)
        if k < 256:
            tk = k
        while k % tk:
            tk //= 2
        out[op] = (t_m, tn, tk)
    out["silu_chunk"] = min(STANDARD_TILE_PROFILE["silu_chunk"], model.ffn_dim // tp)
    return out


def layer_weight_bytes(model: ModelConfig) -> int:
    d, f = model.hidden_dim, model.ffn_dim
    lin = d * model.qkv_dim + d * d + d * model.gate_up_dim + f * d
    norms = 2 * d + 2 * model.head_dim  # rms1/rms2 gammas + q_norm/k_norm
    return (lin + norms) * model.dtype_bytes


def decode_step_bytes(model: ModelConfig, batch: int, ctx: int,
                      vocab: int, layers: int | None = None) -> dict:
    """Algorithmic HBM bytes of one decode step.

    weights (every layer + final norm + LM head) + KV read of ``ctx`` cached
    tokens per sequence.  Activations are ignored (they are <0.1% and stay
    in L2).
    """
    L = model.num_layers if layers is None else layers
    dt = model.dtype_bytes
    w = L * layer_weight_bytes(model) + model.hidden_dim * dt \
        + vocab * model.hidden_dim * dt
    kv = batch * ctx * L * 2 * model.kv_heads * model.head_dim * dt
    return {"weights": w, "kv": kv, "total": w + kv}
