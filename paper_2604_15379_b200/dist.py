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


def allreduce_bytes_per_step(spec, batch: int, dtype_bytes: int = 2) -> dict:
    """Two row-parallel allreduces of [B, hidden] per layer."""
    per = batch * spec.hidden * dtype_bytes
    return {"calls": 2 * spec.layers, "bytes_per_call": per,
            "bytes_per_step": 2 * spec.layers * per}
