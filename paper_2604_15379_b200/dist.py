"""Multi-GPU plumbing: one process per GPU over torch.distributed.

Two things live here:

* replica helpers used by ``bench.py --gpus N`` today (every rank decodes its
  own batch; the job's time is the max over ranks);
* the Megatron-style tensor-parallel partition of one Qwen3 decode step
  (SURVEY.md section 8(e)): column-parallel QKV by kv-head groups and
  gate/up by FFN columns, row-parallel O and down (their partial sums are
  the two per-layer allreduces), vocab-parallel LM head with a (max, index)
  all-gather.  :func:`tp_plan` is the host-side plan the device TP path
  consumes; ``tests/test_dist_gloo.py`` proves the decomposition equals the
  unsharded step on CPU with the gloo backend (world size 2).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch
import torch.distributed as dist


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str):
    rank, world, local = env_rank()
    if world > 1 and not dist.is_initialized():
        dist.init_process_group(backend)
    return rank, world, local


def max_over_ranks(x: float, device="cpu") -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


@dataclass(frozen=True)
class TPPlan:
    """Per-rank slices of one Qwen3 decode step under tensor parallelism."""

    tp: int
    rank: int
    q_heads: range          # query heads owned (follow the kv-head groups)
    kv_heads: range
    ffn: range              # gate/up output columns == down input rows
    vocab: range
    hidden: int

    @property
    def q_cols(self):
        return self.q_heads

    def describe(self):
        return {"tp": self.tp, "rank": self.rank,
                "q_heads": [self.q_heads.start, self.q_heads.stop],
                "kv_heads": [self.kv_heads.start, self.kv_heads.stop],
                "ffn": [self.ffn.start, self.ffn.stop],
                "vocab": [self.vocab.start, self.vocab.stop]}


def tp_plan(spec, tp: int, rank: int) -> TPPlan:
    """Megatron partition: kv heads (with their q-head groups), FFN and vocab
    split evenly; the hidden dimension is replicated."""
    if spec.kv_heads % tp or spec.ffn % tp or spec.vocab % tp:
        raise ValueError(f"TP={tp} does not divide kv_heads/ffn/vocab of {spec}")
    kv = spec.kv_heads // tp
    f = spec.ffn // tp
    v = spec.vocab // tp
    g = spec.group
    return TPPlan(tp, rank, range(rank * kv * g, (rank + 1) * kv * g),
                  range(rank * kv, (rank + 1) * kv), range(rank * f, (rank + 1) * f),
                  range(rank * v, (rank + 1) * v), spec.hidden)


def shard_spec(spec, tp: int):
    """The Qwen3Spec of one rank's shard (hidden / head_dim replicated)."""
    from dataclasses import replace
    plan = tp_plan(spec, tp, 0)
    return replace(spec, ffn=len(plan.ffn), q_heads=len(plan.q_heads),
                   kv_heads=len(plan.kv_heads), vocab=len(plan.vocab))


def shard_weights(w, tp: int, rank: int):
    """Rank ``rank``'s slices of the canonical weights (tp_plan): QKV rows of
    its kv-head groups, O columns of its q heads, gate/up rows and down
    columns of its FFN range, LM-head rows of its vocab range; embedding and
    norm gammas replicated."""
    from .weights import Qwen3Weights
    sp = w.spec
    plan = tp_plan(sp, tp, rank)
    hd = sp.head_dim
    qs = slice(plan.q_heads.start * hd, plan.q_heads.stop * hd)
    ks = slice(plan.kv_heads.start * hd, plan.kv_heads.stop * hd)
    fs = slice(plan.ffn.start, plan.ffn.stop)
    layers = []
    for L in w.layers:
        layers.append({"q": L["q"][qs].contiguous(), "k": L["k"][ks].contiguous(),
                       "v": L["v"][ks].contiguous(), "o": L["o"][:, qs].contiguous(),
                       "gate": L["gate"][fs].contiguous(), "up": L["up"][fs].contiguous(),
                       "down": L["down"][:, fs].contiguous(),
                       **{k: L[k] for k in ("q_norm", "k_norm", "in_norm", "post_norm")}})
    return Qwen3Weights(shard_spec(sp, tp), w.embed, w.final_norm,
                        w.lm_head[plan.vocab.start:plan.vocab.stop].contiguous(), layers)


def connect_local(mks):
    """Join the Megakernels of one TP group living in this process (same
    GPU, or GPUs with peer access): every rank gets every rank's exchange
    region pointer (mk_tp_init)."""
    bases = [mk.tp_region for mk in mks]
    for mk in mks:
        mk.tp_connect(bases)


def connect_dist(mk):
    """Join a TP group of one process per GPU (torch.distributed over
    NCCL/gloo for the bootstrap only): CUDA IPC handles of the exchange
    regions are all-gathered, each peer's region opened, mk_tp_init."""
    import ctypes as C
    from . import _lib as L
    lib = L.load()
    h = (C.c_uint8 * 64)()
    L.check(lib.mk_ipc_export(C.c_void_p(mk.tp_region), h))
    handles = [None] * dist.get_world_size()
    dist.all_gather_object(handles, bytes(h))
    bases = []
    for q, hb in enumerate(handles):
        if q == mk.tp[0]:
            bases.append(mk.tp_region)
            continue
        buf = (C.c_uint8 * 64).from_buffer_copy(hb)
        ptr = C.c_void_p()
        L.check(lib.mk_ipc_import(mk.device, buf, C.byref(ptr)))
        mk.tp_opened.append(ptr.value)
        bases.append(ptr.value)
    mk.tp_connect(bases)


def allreduce_bytes_per_step(spec, batch: int, dtype_bytes: int = 2) -> dict:
    """Two row-parallel allreduces of [B, hidden] per layer."""
    per = batch * spec.hidden * dtype_bytes
    return {"calls": 2 * spec.layers, "bytes_per_call": per,
            "bytes_per_step": 2 * spec.layers * per}
