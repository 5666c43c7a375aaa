"""Hierarchical task graphs for one Qwen3 decode step (drop-in for ``chipletsim.taskgraph``).

A task occupies one hardware scope (wavefront / CU=SM / chiplet=die /
device), waits on events and signals exactly one event; an event fires once
``required_count`` completions arrived (ref
``/root/reference/pkg/src/chipletsim/taskgraph.py:1-18``).

:func:`build_decoder_layer` emits the same graph as the reference -- same task
ids, levels, op kinds, die bindings, gemm/tile shapes, wait/signal events,
required counts and downstream lists, hence the same ``graph_to_json`` bytes
(pinned by ``tests/test_api_parity.py`` against fixtures generated from the
reference).  It is re-expressed here as a table of stages driving two
decomposition rules:

* ``standard`` (die-unaware): every linear op shatters into CU tile tasks
  ``L{l}.{op}.t{m*n_tiles+n}``; SiLU is a separate wavefront-task group.
* ``chiplet`` (die-aware): every linear op becomes one die task per die,
  ``L{l}.{op}.x{die}``, an N-split of the output columns; SiLU is fused into
  the gate/up die task.

What this module adds over the reference is :attr:`TaskGraph.buffers`, the
named activation/weight regions of each layer, which the device lowering
(:mod:`.lowering`) maps onto real HBM allocations.  It is not part of the
JSON export, so parity is unaffected.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

from .machine import MachineConfig, ModelConfig
from .traversal import GemmPartition


class GraphError(ValueError):
    """Graph construction or validation failure (ref taskgraph.py:30)."""


class TaskLevel(Enum):
    WAVEFRONT = "wavefront"
    CU = "cu"
    CHIPLET = "chiplet"
    DEVICE = "device"


def worker_multiplicity(level: TaskLevel, machine: MachineConfig) -> int:
    """Workers one task of ``level`` occupies (ref taskgraph.py:41-47)."""
    return {
        TaskLevel.WAVEFRONT: 1,
        TaskLevel.CU: 1,
        TaskLevel.CHIPLET: machine.workers_per_xcd,
        TaskLevel.DEVICE: machine.workers_per_xcd * machine.num_xcds,
    }[level]


class OpKind(Enum):
    RMS_NORM = "rms_norm"
    QKV_PROJ = "qkv_proj"
    ATTN_PARTIAL = "attn_partial"
    ATTN_REDUCE = "attn_reduce"
    O_PROJ_RESIDUAL = "o_proj_residual"
    GATE_UP_SILU = "gate_up_silu"
    SILU = "silu"
    DOWN_PROJ_RESIDUAL = "down_proj_residual"


LINEAR_OPS = (OpKind.QKV_PROJ, OpKind.O_PROJ_RESIDUAL, OpKind.GATE_UP_SILU,
              OpKind.DOWN_PROJ_RESIDUAL)


@dataclass(frozen=True)
class GemmWork:
    """A die's whole GEMM partition, run cooperatively by the die's workers."""

    partition: GemmPartition
    extra_read_bytes: tuple = ()


@dataclass(frozen=True)
class GemmTileWork:
    """One output tile of a device-wide GEMM (standard-mode CU task)."""

    partition: GemmPartition
    m_idx: int
    n_idx: int
    extra_read_bytes: tuple = ()


@dataclass(frozen=True)
class ElementwiseWork:
    reads: tuple = ()
    writes: tuple = ()


@dataclass(frozen=True)
class OpaqueWork:
    """Dependency-only payload in the reference; the device gives it a body."""


@dataclass(frozen=True)
class Task:
    id: str
    level: TaskLevel
    op_kind: OpKind
    wait_events: tuple = ()
    signal_event: str | None = None
    xcd_binding: int | None = None
    gemm_shape: tuple | None = None
    tile_shape: tuple | None = None
    work: object = OpaqueWork()
    stage: int = -1
    flops: int = 0


@dataclass(frozen=True)
class Event:
    id: str
    required_count: int
    downstream_tasks: tuple = ()


@dataclass(frozen=True)
class StageRecord:
    index: int
    layer: int
    name: str
    op_kind: OpKind
    task_ids: tuple
    event_id: str
    flops: int


@dataclass(frozen=True)
class TaskGraph:
    tasks: tuple
    events: dict
    stages: tuple
    machine: MachineConfig
    model: ModelConfig | None
    batch: int
    mode: str
    op_counts: tuple = ()
    notes: tuple = ()
    # new: per-layer named regions {name: (offset, nbytes)}, one dict per layer
    buffers: tuple = field(default=(), compare=False)

    def task_by_id(self, task_id: str) -> Task:
        idx = self.__dict__.get("_by_id")
        if idx is None:
            idx = {t.id: t for t in self.tasks}
            object.__setattr__(self, "_by_id", idx)
        return idx[task_id]


def adopt_graph(g) -> "TaskGraph":
    """This module's TaskGraph for ``g``, which may have been built by the
    reference package itself (``chipletsim``, same field names, its own enum
    classes: ref taskgraph.py:46-145).  Enum members are re-keyed by value;
    payloads are used by attribute, so they pass through unchanged.  The
    device lowering calls this first, so a graph built by either builder
    lowers to the same descriptors."""
    if isinstance(g, TaskGraph) and all(isinstance(t.op_kind, OpKind) for t in g.tasks):
        return g
    tasks = tuple(Task(t.id, TaskLevel(t.level.value), OpKind(t.op_kind.value),
                       tuple(t.wait_events), t.signal_event, t.xcd_binding,
                       t.gemm_shape, t.tile_shape, t.work, t.stage, t.flops)
                  for t in g.tasks)
    events = {k: Event(e.id, e.required_count, tuple(e.downstream_tasks))
              for k, e in g.events.items()}
    stages = tuple(StageRecord(s.index, s.layer, s.name, OpKind(s.op_kind.value),
                               tuple(s.task_ids), s.event_id, s.flops) for s in g.stages)
    return TaskGraph(tasks, events, stages, g.machine, g.model, g.batch, g.mode,
                     tuple(g.op_counts), tuple(g.notes), tuple(getattr(g, "buffers", ())))


STANDARD_TILE_PROFILE = {
    OpKind.QKV_PROJ: (16, 64, 256),
    OpKind.O_PROJ_RESIDUAL: (16, 16, 256),
    OpKind.GATE_UP_SILU: (16, 128, 256),
    OpKind.DOWN_PROJ_RESIDUAL: (16, 16, 256),
    "silu_chunk": 128,
}

DEFAULT_CHIPLET_TILE = (16, 64, 256)

_LINE_ALIGN = 4096


def _cdiv(a: int, b: int) -> int:
    return (a + b - 1) // b


class _Regions:
    """4 KiB-aligned bump allocation of abstract byte offsets."""

    def __init__(self):
        self.top = 0

    def __call__(self, nbytes: int) -> int:
        at = self.top
        self.top += _cdiv(nbytes, _LINE_ALIGN) * _LINE_ALIGN
        return at


@dataclass
class _Proto:
    """A task before its stage attaches events."""

    id: str
    level: TaskLevel
    xcd_binding: int | None = None
    gemm_shape: tuple | None = None
    tile_shape: tuple | None = None
    work: object = OpaqueWork()
    flops: int = 0


class _Graph:
    def __init__(self, machine, model, batch, mode, dtype_bytes):
        self.machine, self.model = machine, model
        self.batch, self.mode = batch, mode
        self.dt = dtype_bytes
        self.tasks, self.stages, self.op_counts, self.notes = [], [], [], []
        self.required = {}
        self.waiters = {}
        self.regions = _Regions()
        self.buffers = []

    def stage(self, layer, name, kind, protos, after, flops):
        ev = f"e.L{layer}.{name}"
        idx = len(self.stages)
        waits = (after,) if after else ()
        for p in protos:
            self.tasks.append(Task(
                id=p.id, level=p.level, op_kind=kind, wait_events=waits,
                signal_event=ev, xcd_binding=p.xcd_binding,
                gemm_shape=p.gemm_shape, tile_shape=p.tile_shape,
                work=p.work, stage=idx, flops=p.flops))
            for w in waits:
                self.waiters.setdefault(w, []).append(p.id)
        self.required[ev] = len(protos)
        self.stages.append(StageRecord(idx, layer, name, kind,
                                       tuple(p.id for p in protos), ev, flops))
        return ev

    def done(self) -> TaskGraph:
        events = {e: Event(e, n, tuple(self.waiters.get(e, ())))
                  for e, n in self.required.items()}
        return TaskGraph(tuple(self.tasks), events, tuple(self.stages),
                         self.machine, self.model, self.batch, self.mode,
                         tuple(self.op_counts), tuple(self.notes),
                         tuple(self.buffers))


def _require_divides(op, what, dim, tile, allow_padding):
    if not allow_padding and dim % tile:
        raise GraphError(f"{op.value}: tile does not divide {what} "
                         f"({dim} % {tile}) and padding is disabled")


def _linear_protos(g: _Graph, layer, name, op, M, K, N, tile, w_at, a_at,
                   o_at, extra=(), fused=False, allow_padding=True):
    """CU tiles (standard) or one die task per die (chiplet) for one GEMM."""
    t_m, t_n, t_k = tile
    flops = 2 * M * K * N
    dt = g.dt
    if g.mode == "standard":
        _require_divides(op, "M", M, t_m, allow_padding)
        _require_divides(op, "N", N, t_n, allow_padding)
        whole = GemmPartition(M=M, K=K, N_local=N, T_M=t_m, T_N=t_n, T_K=t_k,
                              weight_base=w_at, act_base=a_at, out_base=o_at,
                              dtype_bytes=dt)
        mt, nt = whole.m_tiles, whole.n_tiles
        per_tile = flops // (mt * nt)
        protos = []
        for flat in range(mt * nt):
            m, n = divmod(flat, nt)
            rides = tuple(extra) if flat == 0 else ()
            protos.append(_Proto(
                id=f"L{layer}.{name}.t{flat}", level=TaskLevel.CU,
                gemm_shape=(M, K, N), tile_shape=tile,
                work=GemmTileWork(whole, m, n, rides), flops=per_tile))
        return protos, flops

    dies = g.machine.num_xcds
    if N % dies:
        raise GraphError(f"{op.value}: N={N} is not divisible across "
                         f"{dies} XCDs")
    n_loc = N // dies
    _require_divides(op, "M", M, t_m, allow_padding)
    _require_divides(op, "N_local", n_loc, t_n, allow_padding)
    if fused:
        _require_divides(op, "N_local/2", n_loc // 2, t_n, allow_padding)
    width = n_loc // 2 if fused else n_loc
    protos = []
    for x in range(dies):
        part = GemmPartition(
            M=M, K=K, N_local=n_loc, T_M=t_m, T_N=t_n, T_K=t_k,
            weight_base=w_at + x * K * n_loc * dt, act_base=a_at,
            out_base=o_at + x * M * width * dt, dtype_bytes=dt,
            fused_halves=fused)
        share = tuple((base + x * (nb // dies), nb // dies)
                      for base, nb in extra)
        protos.append(_Proto(
            id=f"L{layer}.{name}.x{x}", level=TaskLevel.CHIPLET,
            xcd_binding=x, gemm_shape=(M, K, N), tile_shape=tile,
            work=GemmWork(part, share), flops=flops // dies))
    return protos, flops


def _tile_profile(mode, overrides):
    if mode == "standard":
        prof = dict(STANDARD_TILE_PROFILE)
    else:
        prof = {op: DEFAULT_CHIPLET_TILE for op in LINEAR_OPS}
        prof["silu_chunk"] = STANDARD_TILE_PROFILE["silu_chunk"]
    prof.update(overrides or {})
    return prof


# per-layer regions in the reference's allocation order (taskgraph.py:398-411)
def _layer_regions(model: ModelConfig, B: int, dt: int):
    d, f = model.hidden_dim, model.ffn_dim
    return (
        ("w_qkv", d * model.qkv_dim * dt),
        ("w_o", d * d * dt),
        ("w_gate_up", d * model.gate_up_dim * dt),
        ("w_down", f * d * dt),
        ("gamma1", d * dt),
        ("gamma2", d * dt),
        ("normed1", B * d * dt),
        ("qkv_out", B * model.qkv_dim * dt),
        ("attn_out", B * d * dt),
        ("x_mid", B * d * dt),
        ("normed2", B * d * dt),
        ("gu_out", B * model.gate_up_dim * dt),
        ("silu_out", B * f * dt),
        ("x_out", B * d * dt),
    )


def build_decoder_layer(model: ModelConfig, machine: MachineConfig, mode: str,
                        batch: int, tile_overrides: dict | None = None,
                        layers: int = 1, allow_padding: bool = True
                        ) -> TaskGraph:
    """``layers`` chained Qwen3 decode layers (ref taskgraph.py:355-526).

    Per layer: rms1 -> qkv -> attn_partial x kv_heads -> attn_reduce x
    kv_heads -> o_proj(+residual) -> rms2 -> gate_up(+SiLU in chiplet mode)
    -> [silu, standard mode only] -> down(+residual); layer l+1's rms1 waits
    on layer l's down event.
    """
    if mode not in ("standard", "chiplet"):
        raise GraphError(f"unknown mode {mode!r}")
    if batch < 1:
        raise GraphError("batch must be at least 1")
    if layers < 1:
        raise GraphError("layers must be at least 1")
    if machine.num_xcds <= 0:
        raise GraphError("machine has no XCDs")

    prof = _tile_profile(mode, tile_overrides)
    g = _Graph(machine, model, batch, mode, model.dtype_bytes)
    B, dt = batch, model.dtype_bytes
    d, f = model.hidden_dim, model.ffn_dim
    fused = mode == "chiplet"

    x_in = g.regions(B * d * dt)
    after = None
    for L in range(layers):
        r = {name: (g.regions(n), n) for name, n in _layer_regions(model, B, dt)}
        r["x_in"] = (x_in, B * d * dt)
        g.buffers.append(r)
        at = {k: v[0] for k, v in r.items()}
        counts = []

        def norm(name, src, dst, gamma, after):
            p = _Proto(id=f"L{L}.{name}.t0", level=TaskLevel.CU,
                       work=ElementwiseWork(
                           reads=((src, B * d * dt), (gamma, d * dt)),
                           writes=((dst, B * d * dt),)),
                       flops=4 * B * d)
            counts.append((name, 1))
            return g.stage(L, name, OpKind.RMS_NORM, [p], after, 4 * B * d)

        def linear(name, op, K, N, w, a, o, extra=(), fuse=False):
            protos, fl = _linear_protos(g, L, name, op, B, K, N, prof[op],
                                        w, a, o, extra, fuse, allow_padding)
            counts.append((name, len(protos)))
            return g.stage(L, name, op, protos, after, fl)

        def opaque(name, op):
            protos = [_Proto(id=f"L{L}.{name}.t{i}", level=TaskLevel.CU)
                      for i in range(model.kv_heads)]
            counts.append((name, len(protos)))
            return g.stage(L, name, op, protos, after, 0)

        after = norm("rms1", at["x_in"], at["normed1"], at["gamma1"], after)
        after = linear("qkv", OpKind.QKV_PROJ, d, model.qkv_dim,
                       at["w_qkv"], at["normed1"], at["qkv_out"])
        after = opaque("attn_partial", OpKind.ATTN_PARTIAL)
        after = opaque("attn_reduce", OpKind.ATTN_REDUCE)
        after = linear("o_proj", OpKind.O_PROJ_RESIDUAL, d, d, at["w_o"],
                       at["attn_out"], at["x_mid"],
                       extra=((at["x_in"], B * d * dt),))
        after = norm("rms2", at["x_mid"], at["normed2"], at["gamma2"], after)
        after = linear("gate_up", OpKind.GATE_UP_SILU, d, model.gate_up_dim,
                       at["w_gate_up"], at["normed2"],
                       at["silu_out"] if fused else at["gu_out"], fuse=fused)
        if not fused:
            after = _silu_stage(g, L, prof, B, f, at, after, counts)
        after = linear("down", OpKind.DOWN_PROJ_RESIDUAL, f, d, at["w_down"],
                       at["silu_out"], at["x_out"],
                       extra=((at["x_mid"], B * d * dt),))
        g.op_counts.append(tuple(counts))
        x_in = at["x_out"]

    per_layer = len(g.tasks) // layers
    g.notes.append(
        f"{mode} mode: {per_layer} tasks per layer from per-op counts; "
        "the commonly quoted headline totals (1,407 standard / 543 chiplet "
        "per layer) are not reproducible from the per-op counts and are "
        "flagged rather than matched")
    return g.done()


def _silu_stage(g, L, prof, B, f, at, after, counts):
    """Standard mode's separate SiLU wavefront tasks (ref taskgraph.py:476-504)."""
    dt = g.dt
    chunk = prof["silu_chunk"]
    t_m = prof[OpKind.GATE_UP_SILU][0]
    n_chunks = _cdiv(f, chunk)
    gate_half = B * f * dt
    protos, off = [], 0
    for grp in range(_cdiv(B, t_m)):
        rows = min(t_m, B - grp * t_m)
        for j in range(n_chunks):
            cols = min(chunk, f - j * chunk)
            nb = rows * cols * dt
            protos.append(_Proto(
                id=f"L{L}.silu.t{grp * n_chunks + j}",
                level=TaskLevel.WAVEFRONT,
                work=ElementwiseWork(
                    reads=((at["gu_out"] + off, nb),
                           (at["gu_out"] + gate_half + off, nb)),
                    writes=((at["silu_out"] + off, nb),)),
                flops=4 * rows * cols))
            off += nb
    counts.append(("silu", len(protos)))
    return g.stage(L, "silu", OpKind.SILU, protos, after, 4 * B * f)


def build_gemm_graph(machine: MachineConfig, gemm_shape: tuple, tiles: tuple,
                     mode: str, op_kind: OpKind = OpKind.QKV_PROJ,
                     dtype_bytes: int = 2, allow_padding: bool = True
                     ) -> TaskGraph:
    """One GEMM as a graph (ref taskgraph.py:529-552)."""
    if mode not in ("standard", "chiplet"):
        raise GraphError(f"unknown mode {mode!r}")
    M, K, N = gemm_shape
    g = _Graph(machine, None, M, mode, dtype_bytes)
    w = g.regions(K * N * dtype_bytes)
    a = g.regions(M * K * dtype_bytes)
    o = g.regions(M * N * dtype_bytes)
    g.buffers.append({"w": (w, K * N * dtype_bytes),
                      "act": (a, M * K * dtype_bytes),
                      "out": (o, M * N * dtype_bytes)})
    protos, fl = _linear_protos(g, 0, "gemm", op_kind, M, K, N, tiles, w, a, o,
                                allow_padding=allow_padding)
    g.op_counts.append((("gemm", len(protos)),))
    g.stage(0, "gemm", op_kind, protos, None, fl)
    return g.done()


def validate_graph(g: TaskGraph) -> None:
    """Ids unique, events closed and counted, bindings legal, acyclic
    (ref taskgraph.py:555-617)."""
    ids = [t.id for t in g.tasks]
    known = set(ids)
    if len(known) != len(ids):
        raise GraphError("duplicate task ids")
    signalled = {}
    for t in g.tasks:
        for e in t.wait_events:
            if e not in g.events:
                raise GraphError(f"task {t.id} waits on unknown event {e}")
        if t.signal_event is not None:
            if t.signal_event not in g.events:
                raise GraphError(
                    f"task {t.id} signals unknown event {t.signal_event}")
            signalled[t.signal_event] = signalled.get(t.signal_event, 0) + 1
        if t.level is TaskLevel.CHIPLET:
            if t.xcd_binding is None:
                raise GraphError(f"chiplet task {t.id} has no XCD binding")
            if not (0 <= t.xcd_binding < g.machine.num_xcds):
                raise GraphError(
                    f"chiplet task {t.id} bound to XCD {t.xcd_binding}, "
                    f"machine has {g.machine.num_xcds}")
        elif t.xcd_binding is not None:
            raise GraphError(f"non-chiplet task {t.id} has an XCD binding")
    for eid, ev in g.events.items():
        n = signalled.get(eid, 0)
        if n != ev.required_count:
            raise GraphError(f"event {eid} requires {ev.required_count} "
                             f"completions but {n} tasks signal it")
        for d in ev.downstream_tasks:
            if d not in known:
                raise GraphError(f"event {eid} releases unknown task {d}")
    _check_acyclic(g)


def _check_acyclic(g: TaskGraph) -> None:
    """Iterative DFS over task -> signal event -> waiting task edges."""
    waiting = {}
    for t in g.tasks:
        for e in t.wait_events:
            waiting.setdefault(e, []).append(t.id)
    by_id = {t.id: t for t in g.tasks}
    colour = {}
    for root in by_id:
        if colour.get(root):
            continue
        path = [root]
        colour[root] = 1
        iters = [iter(waiting.get(by_id[root].signal_event, ()))
                 if by_id[root].signal_event else iter(())]
        while iters:
            nxt = next(iters[-1], None)
            if nxt is None:
                colour[path.pop()] = 2
                iters.pop()
                continue
            c = colour.get(nxt, 0)
            if c == 1:
                cyc = path[path.index(nxt):] + [nxt]
                raise GraphError("cycle detected: " + " -> ".join(cyc))
            if c == 0:
                colour[nxt] = 1
                path.append(nxt)
                sig = by_id[nxt].signal_event
                iters.append(iter(waiting.get(sig, ())) if sig else iter(()))


def cross_chiplet_event_reduction(g_standard: TaskGraph,
                                  g_chiplet: TaskGraph) -> float:
    """Mean ratio of completion signals per linear stage (ref taskgraph.py:620-644)."""
    if (g_standard.machine, g_standard.model, g_standard.batch) != (
            g_chiplet.machine, g_chiplet.model, g_chiplet.batch):
        raise GraphError("graphs built from different configs")
    other = {(s.layer, s.name): s for s in g_chiplet.stages
             if s.op_kind in LINEAR_OPS}
    ratios = []
    for s in g_standard.stages:
        if s.op_kind not in LINEAR_OPS:
            continue
        o = other.get((s.layer, s.name))
        if o is None:
            raise GraphError(f"stage {s.name} missing from second graph")
        ratios.append(len(s.task_ids) / len(o.task_ids))
    if not ratios:
        raise GraphError("no linear stages to compare")
    return sum(ratios) / len(ratios)


def graph_to_json(g: TaskGraph) -> dict:
    """The parity artifact: tasks, sorted events, edges (ref taskgraph.py:647-682)."""
    ev_sorted = sorted(g.events.items())
    tasks = []
    for t in g.tasks:
        tasks.append({
            "id": t.id,
            "level": t.level.value,
            "op_kind": t.op_kind.value,
            "xcd": t.xcd_binding,
            "gemm_shape": list(t.gemm_shape) if t.gemm_shape else None,
            "tile_shape": list(t.tile_shape) if t.tile_shape else None,
            "wait_events": list(t.wait_events),
            "signal_event": t.signal_event,
        })
    edges = [[t.id, t.signal_event] for t in g.tasks if t.signal_event]
    for eid, ev in ev_sorted:
        edges.extend([eid, d] for d in ev.downstream_tasks)
    return {
        "schema_version": 1,
        "mode": g.mode,
        "batch": g.batch,
        "tasks": tasks,
        "events": [{"id": eid, "required_count": ev.required_count,
                    "downstream_tasks": list(ev.downstream_tasks)}
                   for eid, ev in ev_sorted],
        "edges": edges,
    }


def graph_to_dot(g: TaskGraph) -> str:
    """One node per stage (ref taskgraph.py:685-698)."""
    out = ["digraph taskgraph {", "  rankdir=TB;"]
    for s in g.stages:
        out.append(f'  "s{s.index}" [shape=box, '
                   f'label="L{s.layer} {s.name}\\n{len(s.task_ids)} tasks"];')
    stage_of_event = {s.event_id: s.index for s in g.stages}
    for s in g.stages:
        head = g.task_by_id(s.task_ids[0])
        out.extend(f'  "s{stage_of_event[e]}" -> "s{s.index}";'
                   for e in head.wait_events if e in stage_of_event)
    out.append("}")
    return "\n".join(out) + "\n"
