"""Device runtime: the B200 replacement of the reference's ``simulate``.

The reference executes a TaskGraph with ``simulate(g, machine, h, *,
traversal, distribution, ...)`` (``runtime.py:253-548``), a Python model of a
persistent kernel.  Here the same graph is lowered (:mod:`.lowering`) and
executed by the real persistent kernel through the C ABI (``include/mk.h``):

    topo = probe()                       # dies from %smid latency clustering
    machine = b200_from_probe(topo.sms_per_die)
    g = build_decoder_layer(model, machine, "chiplet", batch, tiles, layers)
    mk = Megakernel(g, weights, ctx=1024, traversal=..., distribution=...)
    tokens = mk.step()                   # one launch = one decode step

:func:`run` is the drop-in shaped like ``simulate``: it returns a
:class:`DeviceTrace` with the reference counter names (fences,
global_atomics, local_atomics, dispatches, polls) and the event log
(``(step, actor, action, task_id)``, runtime.py:326-477).

There is no CPU path: constructing a Megakernel without a GPU or without
``libmk.so`` raises.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import torch

from . import _lib as L
from .lowering import PIECE_FLOATS, LoweringOptions, lower
from .analytics import UMMA_MIN_BATCH, default_t_m
from .machine import b200_from_probe
from .taskgraph import OpKind, TaskGraph, TaskLevel, adopt_graph
from .traversal import Distribution, Traversal
from .lowering import is_umma_tile
from .weights import (Qwen3Spec, Qwen3Weights, hash_uniform, pack_gate_up_fused,
                      pack_gate_up_umma, pack_tiles, pack_umma, pad_rows, rope_tables)


def probe(device: int = 0) -> L.Topology:
    """Measure the die map of ``device`` (mk_probe)."""
    lib = L.load()
    topo = L.Topology()
    L.check(lib.mk_probe(device, C.byref(topo)))
    return topo


def topology_summary(topo: L.Topology) -> dict:
    return {
        "num_sms": topo.num_sms,
        "num_dies": topo.num_dies,
        "sms_per_die": [topo.sms_per_die[i] for i in range(topo.num_dies)],
        "separation": round(float(topo.separation), 3),
        "near_cycles": round(float(topo.near_cycles), 1),
        "far_cycles": round(float(topo.far_cycles), 1),
    }


def halves_topology(num_sms: int) -> L.Topology:
    """Fallback split by smid halves (used only when the probe cannot
    separate the dies; reported as separation 0)."""
    t = L.Topology()
    t.num_sms = num_sms
    t.num_dies = 2
    t.sms_per_die[0] = num_sms // 2
    t.sms_per_die[1] = num_sms - num_sms // 2
    for i in range(num_sms):
        t.die_of_sm[i] = 0 if i < num_sms // 2 else 1
    return t


def flat_topology(num_sms: int) -> L.Topology:
    t = L.Topology()
    t.num_sms = num_sms
    t.num_dies = 1
    t.sms_per_die[0] = num_sms
    return t


def _graph_tiles(g: TaskGraph):
    tiles = {}
    for t in g.tasks:
        if t.tile_shape and t.op_kind not in tiles:
            tiles[t.op_kind] = tuple(t.tile_shape)
    return tiles


@dataclass
class DeviceState:
    """Every device buffer one graph instance touches (borrowed by the kernel)."""

    spec: Qwen3Spec
    batch: int
    t_max: int
    split: int
    n_splits: int
    embed: torch.Tensor = None
    final_norm: torch.Tensor = None
    lm_packed: torch.Tensor = None
    w_packed: list = field(default_factory=list)
    w_layers: list = field(default_factory=list)
    layers: list = field(default_factory=list)
    k_cache: list = field(default_factory=list)
    v_cache: list = field(default_factory=list)
    x_in0: torch.Tensor = None
    final_normed: torch.Tensor = None
    logits: torch.Tensor = None
    amax_val: torch.Tensor = None
    amax_idx: torch.Tensor = None
    partial: torch.Tensor = None
    kpart: torch.Tensor = None
    tokens: torch.Tensor = None
    out_tokens: torch.Tensor = None
    positions: torch.Tensor = None
    rope_cos: torch.Tensor = None
    rope_sin: torch.Tensor = None
    vocab_pad: int = 0
    page_table: torch.Tensor = None
    fold_norm: bool = False
    ss_in0: torch.Tensor = None


def build_state(g: TaskGraph, weights: Qwen3Weights, t_max: int, lm_tile,
                amax_slots: int, device="cuda", split: int | None = None,
                keep_logits: bool = True, kv_pages: int | None = None,
                allow_fold: bool = True, kv_share: "DeviceState | None" = None) -> DeviceState:
    """Device buffers of one lowered graph.  ``kv_pages``: paged KV -- every
    layer's K and V become pools of ``kv_pages`` pages of ``split`` tokens
    ([pages][kv_heads][split][head_dim]) addressed through a per-row page
    table ([B][t_max / split] int32, Megakernel assigns pages)."""
    g = adopt_graph(g)
    sp = weights.spec
    B = g.batch
    dev = torch.device(device)
    hd = sp.head_dim
    split = split or max(8, 8192 // hd)
    n_splits = (t_max + split - 1) // split
    t_max = n_splits * split          # whole splits: a split's K/V block never leaves its row
    st = DeviceState(sp, B, t_max, split, n_splits)
    w = weights.to(dev)
    tiles = _graph_tiles(g)
    chiplet = g.mode == "chiplet"
    # tcgen05 everywhere: RMSNorms are folded into their consumers' weights
    # (W * gamma, packed below); lowering.lower scales by 1/rms in the
    # epilogue from the sums of squares the residual GEMMs emit
    fold = (allow_fold and os.environ.get("MK_NO_FOLD") is None
            and all(is_umma_tile(tiles[op], op is OpKind.GATE_UP_SILU and chiplet)
                for op in (OpKind.QKV_PROJ, OpKind.O_PROJ_RESIDUAL,
                           OpKind.GATE_UP_SILU, OpKind.DOWN_PROJ_RESIDUAL))
            and is_umma_tile(lm_tile, False))
    st.fold_norm = fold
    fl = (lambda w_, gam: (w_.float() * gam.float()[None, :]).to(w_.dtype)) if fold \
        else (lambda w_, gam: w_)
    X = g.machine.num_xcds
    bf = dict(device=dev, dtype=torch.bfloat16)
    # layers from the graph's stages (a reference-built TaskGraph carries no
    # buffer table: ref taskgraph.py:135-145)
    n_layers = max((s.layer for s in g.stages), default=-1) + 1
    for li in range(n_layers):
        Lw = w.layers[li]
        qkv = torch.cat((Lw["q"], Lw["k"], Lw["v"]), 0)

        def pk(w_, op):
            _, tn, tk = tiles[op]
            return pack_umma(w_, tn, tk) if is_umma_tile(tiles[op], False) else pack_tiles(w_, tn, tk)

        packed = {"qkv": pk(fl(qkv, Lw["in_norm"]), OpKind.QKV_PROJ),
                  "o": pk(Lw["o"], OpKind.O_PROJ_RESIDUAL),
                  "down": pk(Lw["down"], OpKind.DOWN_PROJ_RESIDUAL)}
        gt = tiles[OpKind.GATE_UP_SILU]
        if chiplet:
            if is_umma_tile(gt, True):
                packed["gate_up"] = pack_gate_up_umma(fl(Lw["gate"], Lw["post_norm"]),
                                                      fl(Lw["up"], Lw["post_norm"]), X, gt[2])
            else:
                packed["gate_up"] = pack_gate_up_fused(Lw["gate"], Lw["up"], X, gt[1], gt[2])
        else:
            packed["gate_up"] = pk(fl(torch.cat((Lw["gate"], Lw["up"]), 0), Lw["post_norm"]),
                                   OpKind.GATE_UP_SILU)
        st.w_packed.append(packed)
        st.w_layers.append({k: Lw[k] for k in ("q_norm", "k_norm", "in_norm", "post_norm")})
        st.layers.append({
            "normed1": torch.zeros(B, sp.hidden, **bf),
            "qkv_out": torch.zeros(B, sp.qkv_dim, **bf),
            "attn_out": torch.zeros(B, sp.hidden, **bf),
            "x_mid": torch.zeros(B, sp.hidden, **bf),
            "normed2": torch.zeros(B, sp.hidden, **bf),
            "gu_out": torch.zeros(B, 2 * sp.ffn, **bf) if not chiplet else None,
            "silu_out": torch.zeros(B, sp.ffn, **bf),
            "x_out": torch.zeros(B, sp.hidden, **bf),
            # folded-norm statistics: per (32-column group) sums of squares
            "ss_mid": torch.zeros(sp.hidden // 32, B, device=dev) if fold else None,
            "ss_out": torch.zeros(sp.hidden // 32, B, device=dev) if fold else None,
        })
        kv_shape = (kv_pages, sp.kv_heads, split, hd) if kv_pages else (B, sp.kv_heads, t_max, hd)
        if kv_share is not None:        # another instance's page pools (chunked prefill)
            st.k_cache.append(kv_share.k_cache[li])
            st.v_cache.append(kv_share.v_cache[li])
        else:
            st.k_cache.append(torch.zeros(*kv_shape, **bf))
            st.v_cache.append(torch.zeros(*kv_shape, **bf))
    del w.layers[:]
    _, tn, tk = lm_tile
    if is_umma_tile(lm_tile, False):
        st.vocab_pad = -(-sp.vocab // 256) * 256          # 128-row tiles per die
        st.lm_packed = pack_umma(pad_rows(fl(w.lm_head, w.final_norm), 256), tn, tk)
    else:
        st.vocab_pad = sp.vocab
        st.lm_packed = pack_tiles(w.lm_head, tn, tk)
    st.embed = w.embed
    st.final_norm = w.final_norm
    st.x_in0 = torch.zeros(B, sp.hidden, **bf)
    st.ss_in0 = torch.zeros(1, B, device=dev) if fold else None
    st.final_normed = torch.zeros(B, sp.hidden, **bf)
    st.logits = torch.zeros(B, st.vocab_pad, device=dev, dtype=torch.float32) \
        if keep_logits else None
    st.amax_val = torch.zeros(amax_slots, B, device=dev, dtype=torch.float32)
    st.amax_idx = torch.zeros(amax_slots, B, device=dev, dtype=torch.int32)
    # pieces: n_splits x (8 warps / group) token subsets, each G x (HD + 4)
    st.partial = torch.zeros(B * sp.kv_heads * n_splits * 8 * (hd + 4),
                             device=dev, dtype=torch.float32)
    st.tokens = torch.zeros(B, device=dev, dtype=torch.int32)
    st.out_tokens = torch.zeros(B, device=dev, dtype=torch.int32)
    st.positions = torch.zeros(B, device=dev, dtype=torch.int32)
    st.page_table = torch.zeros(B, n_splits, device=dev, dtype=torch.int32) if kv_pages else None
    cos, sin = rope_tables(hd, sp.rope_theta, t_max)
    st.rope_cos, st.rope_sin = cos.to(dev), sin.to(dev)
    return st


class PagePool:
    """Free list of KV pages (paged KV): pages are handed out in an
    interleaved order, so a row's pages are in general not contiguous."""

    def __init__(self, n_pages: int):
        order = list(range(0, n_pages, 2)) + list(range(1, n_pages, 2))
        self.free = order[::-1]
        self.n_pages = n_pages

    def alloc(self) -> int:
        if not self.free:
            raise L.MkError(L.MK_ERR_CONFIG, "KV page pool exhausted")
        return self.free.pop()

    def release(self, pages):
        self.free.extend(int(p) for p in pages if p >= 0)


class Megakernel:
    """One lowered graph bound to one device: ``step()`` = one decode step."""

    def __init__(self, g: TaskGraph, weights: Qwen3Weights, *, t_max: int,
                 traversal: Traversal = Traversal.M_MAJOR_WINDOWED,
                 distribution: Distribution = Distribution.M_TILE,
                 sched: str = "per_die", topo: L.Topology | None = None,
                 fanout: bool = True, lm_tile=None, device: int = 0,
                 keep_logits: bool = True, watchdog_s: float = 10.0,
                 ksplit: bool = True, fuse_attn_reduce: bool = False,
                 tp: tuple | None = None, ctas: int | None = None,
                 cooperative: bool = True, kv_pages: int | None = None,
                 prefill_for: "Megakernel | None" = None):
        """``tp=(rank, world)``: this rank's shard of a Megatron tensor-
        parallel group (``weights`` are the full model; dist.shard_weights
        slices them); join the group with dist.connect_local /
        dist.connect_dist before the first step.  ``ctas`` (flat scheduler
        only) launches that many CTAs -- several ranks can then share one GPU
        on disjoint SMs (``cooperative=False``: plain launches).
        ``kv_pages``: paged KV cache with a pool of that many pages of one
        attention split (64 tokens on the tensor-core path) per layer; pages
        are assigned as rows advance and returned by release_row().
        ``prefill_for=mk``: a chunked-prefill instance for the paged decode
        instance ``mk`` (same weights, same page pools): its B rows are B
        consecutive prompt tokens of one of mk's sequences (mk.prefill_chunked)."""
        if not torch.cuda.is_available():
            raise RuntimeError("Megakernel needs a CUDA device (no CPU fallback)")
        self.lib = L.load()
        torch.cuda.set_device(device)
        self.device = device
        self.graph = g = adopt_graph(g)
        self.tp = tuple(tp) if tp else (0, 1)
        self.tp_region, self.tp_opened = None, []
        if self.tp[1] > 1:
            from .dist import shard_weights
            weights = shard_weights(weights, self.tp[1], self.tp[0])
        self.spec = weights.spec
        if topo is None:
            topo = probe(device)
        self.topo = topo
        per_die = sched == "per_die"
        if ctas is not None and per_die:
            raise ValueError("ctas: flat scheduler only")
        if per_die:
            workers = g.machine.workers_per_xcd
            n_dies = g.machine.num_xcds
        else:
            workers = (ctas or topo.num_sms) - 1
            n_dies = 1
        if lm_tile is None:
            lm_tile = _default_lm_tile(self.spec, g.batch)
        opts = LoweringOptions(
            sched_mode=L.SCHED_PER_DIE if per_die else L.SCHED_FLAT,
            traversal=traversal, distribution=distribution, workers=workers,
            n_dies=n_dies, fanout=fanout, lm_tile=lm_tile,
            fuse_attn_reduce=fuse_attn_reduce, prefill=prefill_for is not None)
        v_pad = (-(-self.spec.vocab // 256) * 256) if is_umma_tile(lm_tile, False) \
            else self.spec.vocab
        amax_slots = (n_dies * workers) if per_die else v_pad // lm_tile[1]
        if prefill_for is not None:
            if not prefill_for.pool or prefill_for.state.t_max != t_max:
                raise ValueError("chunked prefill needs a paged decode instance with the same t_max")
            kv_pages = prefill_for.pool.n_pages
        self.state = build_state(g, weights, t_max, lm_tile, amax_slots,
                                 device=f"cuda:{device}",
                                 keep_logits=keep_logits, kv_pages=kv_pages,
                                 allow_fold=self.tp[1] == 1,
                                 kv_share=prefill_for.state if prefill_for is not None else None)
        self.prefill_for = prefill_for
        # a prefill instance's page table rows all point at the sequence being
        # prefilled (set per chunk); it allocates nothing itself
        self.pool = PagePool(kv_pages) if (kv_pages and prefill_for is None) else None
        if self.pool:
            self._table = torch.full((g.batch, self.state.n_splits), -1, dtype=torch.int32)
        if per_die and ksplit:
            # K-split pieces: [die][worker][first/last segment][128 x 64] fp32
            self.state.kpart = torch.zeros(n_dies * workers * 2 * PIECE_FLOATS,
                                           device=f"cuda:{device}", dtype=torch.float32)
        opts.ksplit = ksplit
        if self.tp[1] > 1:
            from .lowering import TPLayout
            layout = TPLayout(self.tp[1], g.batch, self.spec.hidden, len(self.state.layers))
            ptr = C.c_void_p()
            L.check(self.lib.mk_tp_alloc(device, layout.nbytes, C.byref(ptr)))
            self.tp_region, self.tp_layout = ptr.value, layout
            opts.tp_rank, opts.tp_world, opts.tp_layout = self.tp[0], self.tp[1], layout
        self.lowered = lower(g, self.spec, self.state, opts)
        run_topo = topo if per_die else flat_topology(topo.num_sms)
        # KV cache row layout the lowered attention reads and appends: the
        # tensor-core path stores every 16-byte chunk of a row XOR-swizzled by
        # (token & 7) (csrc kv_swz); the CUDA-core path stores rows linear.
        self.kv_swizzled = self.lowered.kv_swizzled
        self._pos = torch.zeros(g.batch, dtype=torch.int64)   # host copy of positions
        self._desc = self.lowered.desc()
        h = C.c_void_p()
        L.check(self.lib.mk_create(device, C.byref(self._desc), C.byref(run_topo),
                                   C.byref(h)))
        self.h = h
        if ctas is not None or not cooperative:
            L.check(self.lib.mk_set_grid(self.h, ctas or topo.num_sms, 1 if cooperative else 0))
        L.check(self.lib.mk_set_watchdog(self.h, watchdog_s))
        L.check(self.lib.mk_set_prefetch(self.h, int(os.environ.get("MK_PREFETCH", "0"))))
        self.steps = 0

    # ---- state -----------------------------------------------------------
    def set_tokens(self, tokens):
        self.state.tokens.copy_(torch.as_tensor(tokens, dtype=torch.int32))

    def set_positions(self, positions):
        pos = torch.as_tensor(positions, dtype=torch.int64).reshape(-1).cpu()
        if pos.numel() != self.graph.batch:
            raise ValueError(f"need {self.graph.batch} positions, got {pos.numel()}")
        if int(pos.min()) < 0 or int(pos.max()) >= self.state.t_max:
            raise ValueError(f"positions must lie in [0, t_max={self.state.t_max})")
        self._pos = pos.clone()
        self.state.positions.copy_(pos.to(torch.int32))
        self._ensure_pages(self._pos)

    # ---- paged KV ------------------------------------------------------------
    def _ensure_pages(self, upto):
        """Every row holds pages for tokens [0, upto[b]] (the next append)."""
        if not self.pool:
            return
        S = self.state.split
        dirty = False
        for b in range(self.graph.batch):
            for i in range(int(upto[b]) // S + 1):
                if i < self._table.shape[1] and self._table[b, i] < 0:
                    self._table[b, i] = self.pool.alloc()
                    dirty = True
        if dirty:
            self.state.page_table.copy_(self._table.clamp(min=0))

    def release_row(self, b: int):
        """Sequence in row ``b`` finished: its KV pages go back to the pool and
        the row restarts at position 0 (continuous batching)."""
        if self.pool:
            self.pool.release(self._table[b].tolist())
            self._table[b] = -1
        self._pos[b] = 0
        self.state.positions[b] = 0
        self._ensure_pages(self._pos)

    def page_table(self) -> torch.Tensor:
        """Host copy of the page table ([B][t_max / split], -1 = unassigned)."""
        return self._table.clone() if self.pool else None

    def _logical(self, buf: torch.Tensor, n: int) -> torch.Tensor:
        """[B, kvh, n, hd] logical view (a copy when paged)."""
        if not self.pool:
            return buf[:, :, :n]
        S = self.state.split
        rows = []
        for b in range(self.graph.batch):
            blocks = [buf[int(self._table[b, i])] for i in range(-(-n // S))]
            rows.append(torch.cat(blocks, 1)[:, :n])
        return torch.stack(rows)

    def _store_logical(self, buf: torch.Tensor, x: torch.Tensor):
        """Write [B, kvh, n, hd] into tokens [0, n) of every row."""
        n = x.shape[2]
        if not self.pool:
            buf[:, :, :n] = x
            return
        self._ensure_pages([n - 1] * self.graph.batch)
        S = self.state.split
        for b in range(self.graph.batch):
            for i in range(-(-n // S)):
                c = min(S, n - i * S)
                buf[int(self._table[b, i]), :, :c] = x[b, :, i * S:i * S + c]

    def positions(self) -> torch.Tensor:
        """Host copy of the decode position of every row (the next token's index)."""
        return self._pos.clone()

    # ---- KV cache (canonical layout [B][kv_head][token][head_dim] bf16) ---
    def _kv_view(self, buf: torch.Tensor) -> torch.Tensor:
        """[B, kvh, T, hd] -> [B, kvh, T, hd/8, 8] chunk view."""
        B, H, T, hd = buf.shape
        return buf.view(B, H, T, hd // 8, 8)

    def _swizzle_index(self, n: int, device):
        t = torch.arange(n, device=device).view(n, 1)
        c = torch.arange(self.spec.head_dim // 8, device=device).view(1, -1)
        return (c ^ (t & 7))                       # physical chunk of logical chunk c

    def write_kv(self, layer: int, k: torch.Tensor, v: torch.Tensor, n_tokens: int):
        """Write tokens [0, n_tokens) of canonical K/V ([B, kv_heads, >=n, hd],
        any dtype) into the device cache in the layout the lowered graph reads
        (INTEGRATION.md section 4)."""
        if n_tokens > self.state.t_max:
            raise ValueError(f"{n_tokens} tokens do not fit t_max={self.state.t_max}")
        for src, dst in ((k, self.state.k_cache[layer]), (v, self.state.v_cache[layer])):
            x = src[:, :, :n_tokens].to(dst.device, torch.bfloat16)
            if self.kv_swizzled:
                B, H, n, hd = x.shape
                idx = self._swizzle_index(n, dst.device).view(1, 1, n, hd // 8, 1)
                out = torch.empty_like(x).view(B, H, n, hd // 8, 8)
                out.scatter_(3, idx.expand(B, H, n, hd // 8, 8), x.view(B, H, n, hd // 8, 8))
                x = out.view(B, H, n, hd)
            self._store_logical(dst, x)

    def read_kv(self, layer: int, n_tokens: int):
        """Canonical (un-swizzled) copies of tokens [0, n_tokens) of the cache."""
        out = []
        for buf in (self.state.k_cache[layer], self.state.v_cache[layer]):
            x = self._logical(buf, n_tokens)
            if self.kv_swizzled:
                B, H, n, hd = x.shape
                idx = self._swizzle_index(n, x.device).view(1, 1, n, hd // 8, 1)
                x = torch.gather(x.reshape(B, H, n, hd // 8, 8), 3,
                                 idx.expand(B, H, n, hd // 8, 8)).view(B, H, n, hd)
            out.append(x.clone())
        return tuple(out)

    def fill_kv_random(self, n_tokens: int, seed: int = 99):
        """Perf runs: ``n_tokens`` of synthetic bf16 context per sequence."""
        sp = self.spec
        shape = (self.graph.batch, sp.kv_heads, n_tokens, sp.head_dim)
        for li, (k, v) in enumerate(zip(self.state.k_cache, self.state.v_cache)):
            for j, buf in enumerate((k, v)):
                u = hash_uniform(int(torch.Size(shape).numel()), seed, 2 * li + j, device=buf.device)
                # i.i.d. values: the swizzled layout is a permutation of them
                self._store_logical(buf, ((u * 2 - 1) * 1.7).to(torch.bfloat16).view(shape))
        self.set_positions([n_tokens] * self.graph.batch)

    # ---- execution ---------------------------------------------------------
    def launch(self, stream=None):
        # every row appends its token at its position: refuse before any row
        # would index past the cache (the device also flags it, mk_sync)
        if int(self._pos.max()) >= self.state.t_max:
            raise L.MkError(L.MK_ERR_CONFIG, f"decode position {int(self._pos.max())} "
                            f"reached t_max={self.state.t_max}")
        self._ensure_pages(self._pos)           # paged KV: the page this append lands in
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        L.check(self.lib.mk_step(self.h, C.c_void_p(s.cuda_stream)))
        self._pos += 1                          # the argmax task advances the positions
        self.steps += 1

    def launch_host(self, tokens_in, tokens_out, stream=None):
        """One step through mk_step_tokens: ``tokens_in`` / ``tokens_out`` are
        host int32 tensors [B] (pinned for asynchrony); the copies and the
        launch are queued on ``stream``."""
        if int(self._pos.max()) >= self.state.t_max:
            raise L.MkError(L.MK_ERR_CONFIG, f"decode position {int(self._pos.max())} "
                            f"reached t_max={self.state.t_max}")
        for t in (tokens_in, tokens_out):
            if t is not None and (t.device.type != "cpu" or t.dtype != torch.int32
                                  or t.numel() != self.graph.batch):
                raise ValueError("host int32 tensors of batch size expected")
        self._ensure_pages(self._pos)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        L.check(self.lib.mk_step_tokens(
            self.h, C.c_void_p(s.cuda_stream),
            C.c_void_p(tokens_in.data_ptr() if tokens_in is not None else 0),
            C.c_void_p(tokens_out.data_ptr() if tokens_out is not None else 0)))
        self._pos += 1
        self.steps += 1

    def sync(self):
        L.check(self.lib.mk_sync(self.h))

    def step(self, tokens=None):
        """One decode step; returns the greedy tokens (int32 [B], on device)."""
        if tokens is not None:
            self.set_tokens(tokens)
        self.launch()
        self.sync()
        return self.state.out_tokens.clone()

    def generate(self, prompts, max_new_tokens: int = 1):
        """Device prefill + greedy decode for ragged prompts (one list of
        token ids per row, any lengths >= 1).  Every row starts at position
        0; step t feeds row b its prompt token t while the prompt lasts, then
        its own previous greedy token, so each row's KV context is built on
        the device by the decode kernels themselves.  Returns, per row, the
        ``max_new_tokens`` greedy tokens that follow its prompt."""
        B = self.graph.batch
        if len(prompts) != B or min(len(p) for p in prompts) < 1:
            raise ValueError(f"need {B} non-empty prompts")
        lens = [len(p) for p in prompts]
        total = max(n + max_new_tokens - 1 for n in lens)
        if total > self.state.t_max:
            raise ValueError(f"{total} positions exceed t_max={self.state.t_max}")
        for b in range(B):
            self.release_row(b)
        outs = [[] for _ in range(B)]
        prev = [0] * B
        for t in range(total):
            toks = [prompts[b][t] if t < lens[b] else prev[b] for b in range(B)]
            prev = self.step(toks).cpu().tolist()
            for b in range(B):
                if t >= lens[b] - 1 and len(outs[b]) < max_new_tokens:
                    outs[b].append(prev[b])
        return outs

    def prefill_chunked(self, row: int, prompt, pf: "Megakernel"):
        """Chunked device prefill of sequence ``row``: ``pf`` (an instance
        built with ``prefill_for=self``) decodes pf.batch prompt tokens per
        launch -- its rows are consecutive positions of this one sequence,
        sharing its pages; the KV of the whole prompt lands in this
        instance's page pools.  Afterwards row ``row`` continues at position
        len(prompt); returns the greedy token after the prompt."""
        if pf.prefill_for is not self:
            raise ValueError("pf was not built with prefill_for=self")
        T, C_ = len(prompt), pf.graph.batch
        if T < 1 or T > self.state.t_max:
            raise ValueError("prompt length out of range")
        self.release_row(row)
        self._ensure_pages([T - 1 if b == row else 0 for b in range(self.graph.batch)])
        table = self.state.page_table[row].clone()
        pf.state.page_table.copy_(table.expand(C_, -1))
        nxt = None
        for c0 in range(0, T, C_):
            n = min(C_, T - c0)
            # pad rows repeat the last real token at its position (identical
            # K/V writes); their outputs are ignored
            pos = [c0 + min(r, n - 1) for r in range(C_)]
            toks = [prompt[c0 + min(r, n - 1)] for r in range(C_)]
            pf._pos = torch.tensor(pos, dtype=torch.int64)
            pf.state.positions.copy_(pf._pos.to(torch.int32))
            out = pf.step(toks).cpu().tolist()
            nxt = out[n - 1]
        self._pos[row] = T
        self.state.positions[row] = T
        self._ensure_pages(self._pos)
        return nxt

    def prefill(self, prompts):
        """Build every row's KV context from its prompt on the device;
        returns the greedy token after each prompt."""
        return [o[0] for o in self.generate(prompts, 1)]

    def logits(self):
        lg = self.state.logits
        return None if lg is None else lg[:, :self.spec.vocab]

    def counters(self) -> dict:
        c = L.Counters()
        L.check(self.lib.mk_counters_get(self.h, C.byref(c)))
        return c.as_dict()

    def reset_counters(self):
        L.check(self.lib.mk_counters_reset(self.h))

    def enable_log(self, capacity: int):
        L.check(self.lib.mk_log_enable(self.h, capacity))

    def read_log(self, capacity: int):
        buf = (L.LogRec * capacity)()
        n = self.lib.mk_log_read(self.h, buf, capacity)
        if n < 0:
            L.check(-n)
        return [buf[i] for i in range(min(n, capacity))], n

    def enable_tile_log(self, capacity: int):
        L.check(self.lib.mk_tile_log_enable(self.h, capacity))

    def read_tile_log(self, capacity: int):
        buf = (C.c_int32 * (4 * capacity))()
        n = self.lib.mk_tile_log_read(self.h, buf, capacity)
        if n < 0:
            L.check(-n)
        m = min(n, capacity)
        return [tuple(buf[4 * i:4 * i + 4]) for i in range(m)], n

    def enable_trace(self, units_per_worker: int):
        """Per-unit phase stamps (mk_trace_enable); 0 turns tracing off."""
        L.check(self.lib.mk_trace_enable(self.h, units_per_worker))
        self._trace_cap = units_per_worker

    def read_trace(self):
        """[workers, units_per_worker, 8] uint64 stamps (see include/mk.h)."""
        import numpy as np
        n = self.lowered.n_sched * self.lowered.workers * self._trace_cap * 8
        buf = np.zeros(n, dtype=np.uint64)
        got = self.lib.mk_trace_read(self.h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), n)
        if got < 0:
            L.check(-got)
        return buf.reshape(-1, self._trace_cap, 8)

    def tp_connect(self, peer_bases):
        """mk_tp_init: ``peer_bases[q]`` = rank q's exchange region as
        addressable from this device (own region at index rank)."""
        arr = (C.c_void_p * len(peer_bases))(*peer_bases)
        L.check(self.lib.mk_tp_init(self.h, self.tp[0], self.tp[1], arr))

    def close(self):
        if getattr(self, "h", None):
            self.lib.mk_destroy(self.h)
            self.h = None
        for p in getattr(self, "tp_opened", []):
            self.lib.mk_ipc_close(C.c_void_p(p))
        self.tp_opened = []
        if getattr(self, "tp_region", None):
            self.lib.mk_tp_free(C.c_void_p(self.tp_region))
            self.tp_region = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _default_lm_tile(spec: Qwen3Spec, batch: int, t_m: int | None = None,
                     umma: bool | None = None):
    """LM-head tile: the tcgen05 body (128 x 64, vocab padded to 256) from
    UMMA_MIN_BATCH rows on, else the warp-row GEMV rule of gemv_tiles."""
    if t_m is None:
        t_m = default_t_m(batch) if umma is not False else 16
    rows = min(batch, t_m)
    use = umma if umma is not None else rows >= UMMA_MIN_BATCH
    if use and spec.hidden % 64 == 0:
        return (t_m, 128, 64)
    t_m = min(t_m, 16)
    t_n = 16 if rows <= 4 else 32
    while (spec.vocab // 2) % t_n and t_n > 8:
        t_n //= 2
    t_k = spec.hidden if spec.hidden < 256 else min(8192 // t_n, spec.hidden)
    while spec.hidden % t_k:
        t_k //= 2
    return (t_m, t_n, t_k)


@dataclass
class DeviceTrace:
    """simulate()-shaped result of device runs (ref runtime.py:92-171).

    ``to_json()`` / ``csv_row()`` emit the reference's record and CSV
    columns (``report.py``), so ``comparison_table`` renders device runs."""

    mode: str
    batch: int
    traversal: str
    distribution: str
    steps: int
    fences_issued: int
    global_atomics: int
    local_atomics: int
    poll_count: int
    dispatches: int
    counters: dict
    event_log: tuple
    metrics: object = None
    stage_costs: tuple = ()
    estimated_time_s: float = 0.0
    policy_notes: tuple = ()
    model_fingerprint: tuple | None = None
    fence_flush_lines: int = 0          # a simulator quantity: no device equivalent

    def to_json(self) -> dict:
        from .report import trace_to_json
        return trace_to_json(self)

    def csv_row(self, scenario_id: str) -> str:
        from .report import trace_csv_row
        return trace_csv_row(self, scenario_id)


def run(g: TaskGraph, weights: Qwen3Weights, *, t_max: int, steps: int = 1,
        traversal=Traversal.M_MAJOR_WINDOWED,
        distribution=Distribution.M_TILE, sched: str = "per_die",
        keep_event_log: bool = True, fanout: bool = True,
        topo=None, positions=None, ncu_csv: str | None = None) -> DeviceTrace:
    """Execute ``steps`` decode steps of ``g`` on the GPU (drop-in for simulate).

    ``positions``: the per-row context at the first step (default 0).
    ``ncu_csv``: text of an ``ncu --csv --metrics`` capture of one of these
    launches; its L2 / DRAM counters become the trace's metrics (else the
    step's algorithmic bytes, L2 hit rate NaN)."""
    from . import report
    mk = Megakernel(g, weights, t_max=t_max, traversal=traversal,
                    distribution=distribution, sched=sched, fanout=fanout,
                    topo=topo)
    if positions is not None:
        mk.set_positions(positions)
    ctx0 = float(mk.positions().float().mean())
    cap = 0
    if keep_event_log:
        cap = 4 * (len(mk.lowered.units) * (g.machine.workers_per_xcd + 1)) + 1024
        mk.enable_log(cap)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)]
    for i in range(steps):
        ev[2 * i].record()
        mk.launch()
        ev[2 * i + 1].record()
        mk.sync()
    secs = sum(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(steps)) / 1e3 / max(steps, 1)
    c = mk.counters()
    log = ()
    if keep_event_log:
        recs, _ = mk.read_log(cap)
        log = tuple(device_log_to_reference(mk, recs))
    ctx = int(round(ctx0 + (steps + 1) / 2))        # mean attended context
    metrics = report.metrics_from_ncu(ncu_csv) if ncu_csv else \
        report.metrics_algorithmic(g, ctx, mk.spec.vocab)
    m = g.model
    tr = DeviceTrace(g.mode, g.batch, traversal.value, distribution.value,
                     steps, c["fences"], c["global_atomics"], c["local_atomics"],
                     c["polls"], c["dispatches"], c, log,
                     metrics=metrics, stage_costs=report.stage_costs(g, ctx),
                     estimated_time_s=secs,
                     policy_notes=(f"sched={sched}", f"metrics={metrics.source}",
                                   "time=measured_device_s_per_step",
                                   f"workers_per_die={mk.lowered.workers}"),
                     model_fingerprint=(m.hidden_dim, m.ffn_dim, m.num_layers, m.q_heads, m.kv_heads))
    mk.close()
    return tr


def device_log_to_reference(mk: Megakernel, recs):
    """Device records -> the reference's (time, actor, action, task_id) tuples.

    Dispatch records come from the scheduler CTAs (actor ``sched.x{die}``),
    execution records from workers (``worker.x{die}.w{w}``).  Time is the
    %globaltimer nanosecond stamp (the reference's logical ``step``).
    """
    names = mk.lowered.task_names
    W = mk.lowered.workers
    out = []
    for r in sorted(recs, key=lambda r: (r.t_start, r.kind)):
        if r.kind == 0:
            out.append((int(r.t_start), f"sched.x{-1 - r.worker}", "dispatch",
                        names[r.task]))
        else:
            out.append((int(r.t_start), f"worker.x{r.die}.w{r.worker % W}",
                        "start", names[r.task]))
            out.append((int(r.t_end), f"worker.x{r.die}.w{r.worker % W}",
                        "complete", names[r.task]))
    return out
