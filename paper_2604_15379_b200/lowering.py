"""Host graph compiler: TaskGraph -> flat device descriptor arrays.

Input: a graph from :func:`.taskgraph.build_decoder_layer` (the reference's
topology, ref taskgraph.py:355-526) plus the device buffers of one model
instance.  Output: the arrays of ``mk_graph_desc`` (include/mk.h):

* one ``mk_task`` per graph task, in graph order, with the event it waits
  on, the event it signals and an op parameter block (device pointers,
  shapes, tile, traversal / distribution);
* three appended stages the reference graph lacks (SURVEY.md section 7.3 item
  9): ``final_norm`` -> ``lm_head`` -> ``argmax``, so one launch produces
  greedy token ids;
* the per-scheduler dispatch lists in topological (graph) order: a die task
  goes to its die's list, CU task units go round-robin across dies in graph
  order -- the reference's ``enqueue`` rule (ref runtime.py:301-307);
* event ``required_count`` (ref taskgraph.py:221) and sub-counters for CU
  tasks whose items are fanned out over several workers (attention, norms):
  the fanned task still signals its event exactly once.

The reference work payloads (GemmWork / GemmTileWork / ElementwiseWork) are
mapped to real pointers: weights are packed tile-major per op
(weights.pack_tiles), a die task's slab pointer is the reference's
``weight_base + x*K*N_local*dtype`` (taskgraph.py:330) realised on the packed
tensor, and its output block starts at column ``x*N_local``.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

from . import _lib as L
from .taskgraph import OpKind, TaskGraph, TaskLevel, adopt_graph
from .traversal import Distribution, Traversal


def _cdiv(a, b):
    return (a + b - 1) // b


def is_umma_tile(tile, fused: bool) -> bool:
    """tcgen05 body tiles: 128 weight rows (64+64 for fused gate/up) x 64."""
    _, t_n, t_k = tile
    return t_k == 64 and t_n * (2 if fused else 1) == 128


KSPLIT_MIN_BALANCE = float(os.environ.get("MK_KSPLIT_BALANCE", "0.85"))
# tensor-core attention from this batch on (barrier-free warps: measured
# faster than the CUDA-core split path at every batch 1-64)
ATTN_MMA_MIN_BATCH = int(os.environ.get("MK_ATTN_MMA_MIN_BATCH", "1"))


def gemv_fast_shape(batch_rows: int, rows: int, t_k: int) -> bool:
    """The register-resident GEMV tile shapes (csrc gemm_tile_fast): the only
    CUDA-core shapes with a K-split variant."""
    return ((batch_rows <= 1 and rows == 8 and t_k == 1024)
            or (batch_rows <= 4 and rows == 16 and t_k == 512)
            or (batch_rows <= 8 and rows == 32 and t_k == 256))


def ksplit_pays(tiles: int, workers: int) -> bool:
    """K-split a die task only when whole-tile round-robin ownership
    (schedule(), traversal.py:125-202) would leave the die's workers
    unbalanced: tiles / (rounds * workers) below KSPLIT_MIN_BALANCE.  Whole
    tiles keep the concurrent workers on adjacent weight tiles (one DRAM
    sweep) and need no partial-sum exchange."""
    rounds = _cdiv(tiles, workers)
    return tiles / (rounds * workers) < KSPLIT_MIN_BALANCE


@dataclass
class LoweringOptions:
    sched_mode: int = L.SCHED_PER_DIE
    traversal: Traversal = Traversal.M_MAJOR_WINDOWED
    distribution: Distribution = Distribution.M_TILE
    workers: int = 73              # W per scheduler
    n_dies: int = 2                # schedulers in PER_DIE mode
    fanout: bool = True            # split CU tasks' items over several units
    lm_tile: tuple = (16, 8, 1024)  # (T_M, T_N, T_K) of the appended LM head
    attn_split: int = 64           # tokens per split-KV item
    fuse_norm: bool = True         # RMSNorm folded into the consuming GEMM's
                                   # activation staging when the rows fit
    bypass_noop: bool = True       # consumers of a fused (no-op) norm task wait
                                   # on that task's own predecessor event
    attn_mma: bool = os.environ.get("MK_ATTN_MMA", "1") != "0"
                                   # tensor-core split-KV attention (head_dim 128)
    fuse_attn_reduce: bool = False # last split of a row merges (ATTN_REDUCE no-op);
                                   # measured slower (one warp merges serially)
    ksplit: bool = True            # die tasks: K-split slot ranges per worker
                                   # instead of whole tiles
    prefill: bool = False          # chunked prefill: the rows are consecutive
                                   # tokens of one sequence (attention folds the
                                   # chunk's earlier tokens into its slots)
    tp_rank: int = 0               # tensor parallelism: this
    tp_world: int = 1              # rank of the group; spec / buffers are the
    tp_layout: object = None       # rank's shard (runtime.build_state), TPLayout


@dataclass(frozen=True)
class TPLayout:
    """Byte layout of one rank's exchange region -- identical on every rank,
    so the offsets baked into the descriptors address any rank's region:
    recv[point][world][B][d] fp32 (point 2l = layer l's o_proj, 2l+1 its
    down proj; slot q = rank q's partial), flags[point][world] uint32
    (point 2L = the LM-head argmax), gather[world][B] {float, int32}."""
    world: int
    batch: int
    hidden: int
    layers: int

    @property
    def n_points(self) -> int:
        return 2 * self.layers

    def recv_off(self, point: int) -> int:
        return point * self.world * self.batch * self.hidden * 4

    def slot_off(self, point: int, rank: int) -> int:
        return self.recv_off(point) + rank * self.batch * self.hidden * 4

    def flag_off(self, point: int) -> int:
        return self.recv_off(self.n_points) + point * self.world * 4

    @property
    def argmax_point(self) -> int:
        return self.n_points

    @property
    def gather_off(self) -> int:
        return -(-self.flag_off(self.n_points + 1) // 16) * 16

    @property
    def nbytes(self) -> int:
        return self.gather_off + self.world * self.batch * 8

XS_BYTES = 49152                   # kXsBytes in mk_kernel.cu
PIECE_FLOATS = 128 * 64            # K-split piece: 128 weight rows x 64 batch rows


@dataclass
class Lowered:
    tasks: object
    units: object
    sched_begin: object
    event_required: object
    params: bytes
    event_names: list
    task_names: list
    graph_task_index: list
    n_sub: int
    n_sched: int
    sched_mode: int
    workers: int
    amax_slots: int
    kv_swizzled: bool = False      # KV rows chunk-swizzled (tensor-core attention)
    positions: int = 0             # device pointer of the per-row decode positions
    n_rows: int = 0
    tokens: int = 0                # device pointers of the step's token ids / greedy ids
    out_tokens: int = 0
    keep: list = field(default_factory=list)   # ctypes arrays kept alive

    def desc(self) -> L.GraphDesc:
        pbuf = C.create_string_buffer(self.params, max(1, len(self.params)))
        self.keep.append(pbuf)
        g = L.GraphDesc()
        g.n_tasks = len(self.tasks)
        g.n_events = len(self.event_required)
        g.n_units = len(self.units)
        g.n_sub_ctrs = self.n_sub
        g.n_schedulers = self.n_sched
        g.sched_mode = self.sched_mode
        g.workers_per_sched = self.workers
        g.param_bytes = len(self.params)
        g.tasks = C.cast(self.tasks, C.c_void_p)
        g.event_required = C.cast(self.event_required, C.c_void_p)
        g.units = C.cast(self.units, C.c_void_p)
        g.sched_begin = C.cast(self.sched_begin, C.c_void_p)
        g.params = C.cast(pbuf, C.c_void_p)
        g.positions = self.positions
        g.n_rows = self.n_rows
        g.tokens = self.tokens
        g.out_tokens = self.out_tokens
        return g


class _Blob:
    def __init__(self):
        self.data = bytearray()

    def add(self, struct) -> int:
        off = len(self.data)
        self.data += bytes(struct)
        while len(self.data) % 8:
            self.data += b"\0"
        return off


class _Off(int):
    """A byte offset standing in for a pointer (MK_EPI_PARTIAL's y)."""


def _ptr(t, elem_offset=0):
    if t is None:
        return None
    if isinstance(t, _Off):
        return int(t) + elem_offset * 4
    return t.data_ptr() + elem_offset * t.element_size()


def lower(g: TaskGraph, spec, bufs, opts: LoweringOptions) -> Lowered:
    """Lower ``g`` against device buffers ``bufs`` (a runtime.DeviceState).
    ``g`` may come from this package's builder or the reference's."""
    g = adopt_graph(g)
    B = g.batch
    d, F, hd = spec.hidden, spec.ffn, spec.head_dim
    per_die = opts.sched_mode == L.SCHED_PER_DIE
    n_sched = opts.n_dies if per_die else 1
    if not per_die:
        for t in g.tasks:
            if t.level is TaskLevel.CHIPLET and t.xcd_binding != 0:
                raise ValueError("the flat scheduler runs die-unaware graphs "
                                 "(standard mode or a 1-die machine)")
    blob = _Blob()
    event_names = list(g.events)
    ev_index = {e: i for i, e in enumerate(event_names)}
    required = [g.events[e].required_count for e in event_names]
    tasks, names, gidx = [], [], []
    units_by_sched = [[] for _ in range(n_sched)]
    rr = [0]
    n_sub = [0]
    total_workers = opts.workers * n_sched
    trav = L.TRAV_M_MAJOR if opts.traversal is Traversal.M_MAJOR_WINDOWED \
        else L.TRAV_N_MAJOR
    dist = L.DIST_M_SPLIT if opts.distribution is Distribution.M_SPLIT \
        else L.DIST_M_TILE

    def add_task(name, graph_i, op, level, die, wait, signal, param_off,
                 layer, n_items=1, n_units=1):
        t = L.Task()
        t.op, t.level = op, level
        t.die = -1 if die is None else die
        t.wait0 = -1 if wait is None else ev_index[wait]
        t.wait1 = -1
        t.signal = -1 if signal is None else ev_index[signal]
        n_units = max(1, min(n_units, n_items)) if opts.fanout else 1
        t.n_items, t.n_units = n_items, n_units
        t.sub_ctr = -1
        if n_units > 1:
            t.sub_ctr = n_sub[0]
            n_sub[0] += 1
        t.param_off, t.layer, t.graph_index = param_off, layer, graph_i
        ti = len(tasks)
        tasks.append(t)
        names.append(name)
        gidx.append(graph_i)
        if level == L.LEVEL_CHIPLET:
            units_by_sched[die if per_die else 0].append((ti, 0, 0))
        else:
            for u in range(n_units):
                ib = u * n_items // n_units
                ie = (u + 1) * n_items // n_units
                s = (rr[0] % n_sched) if per_die else 0
                rr[0] += 1
                units_by_sched[s].append((ti, ib, ie))
        return ti

    def stages(M, K, tile):
        return min(tile[0], M) * K * 2 <= XS_BYTES

    def gemm_params(w, x, y, res, M, K, N, tile, ldx, ldy, ldres, col0, epi,
                    xcd, tm=-1, tn=-1, amax_base=0, gamma=None, y_cols=None,
                    ksplit=False, ss_in=None, ss_out=None):
        p = L.GemmParams()
        if ss_in is not None:          # RMSNorm folded into these weights
            p.ss_in, p.ss_nparts = _ptr(ss_in[0]), ss_in[1]
            p.norm_eps = spec.eps
        p.ss_out = _ptr(ss_out)
        umma = is_umma_tile(tile, epi == L.EPI_SILU)
        rows = tile[1] * (2 if epi == L.EPI_SILU else 1)
        if ksplit and not ksplit_pays(_cdiv(M, tile[0]) * (N // rows), opts.workers):
            ksplit = False
        if ksplit and not umma and not gemv_fast_shape(min(tile[0], M), rows, tile[2]):
            ksplit = False
        if ksplit:
            p.ksplit = 1
            p.tile_ctr0 = n_sub[0]
            n_sub[0] += _cdiv(M, tile[0]) * (N // rows)
            p.piece_floats = PIECE_FLOATS
            p.kpart = _ptr(bufs.kpart, xcd * opts.workers * 2 * PIECE_FLOATS)
        p.body = L.BODY_UMMA if umma else L.BODY_GEMV
        p.stage_x = 0 if umma else (1 if stages(M, K, tile) else 0)
        p.y_cols = y_cols if y_cols is not None else (1 << 30)
        if gamma is not None:
            assert p.stage_x
            p.norm_gamma = _ptr(gamma)
            p.norm_eps = spec.eps
        p.w, p.x, p.y, p.res = w, x, y, res
        p.amax_val = _ptr(bufs.amax_val)
        p.amax_idx = _ptr(bufs.amax_idx)
        p.M, p.K, p.N = M, K, N
        p.T_M, p.T_N, p.T_K = tile
        p.ldx, p.ldy, p.ldres, p.y_col0 = ldx, ldy, ldres, col0
        p.epilogue, p.traversal, p.distribution, p.xcd = epi, trav, dist, xcd
        p.tile_m, p.tile_n = tm, tn
        p.amax_base, p.amax_stride = amax_base, B
        return blob.add(p)

    def norm_params(layer_bufs, x, gamma, y, embed=False, fused=False, ss_out=None):
        p = L.NormParams()
        p.fused = 1 if fused else 0
        p.ss_out = _ptr(ss_out)
        p.x, p.gamma, p.y = _ptr(x), _ptr(gamma), _ptr(y)
        if embed:
            p.embed = _ptr(bufs.embed)
            p.tokens = _ptr(bufs.tokens)
            p.x_store = _ptr(bufs.x_in0)
        p.M, p.d, p.eps = B, d, spec.eps
        return blob.add(p)

    def attn_params(layer, h, out=None, fuse=False, reduce_noop=False):
        lb = bufs.layers[layer]
        p = L.AttnParams()
        p.fuse_reduce = 1 if reduce_noop else 0
        if fuse and fused_reduce:
            p.fuse_reduce = 1
            p.red_ctr0 = n_sub[0]
            n_sub[0] += B
        p.qkv = _ptr(lb["qkv_out"])
        p.q_gamma = _ptr(bufs.w_layers[layer]["q_norm"])
        p.k_gamma = _ptr(bufs.w_layers[layer]["k_norm"])
        p.k_cache, p.v_cache = _ptr(bufs.k_cache[layer]), _ptr(bufs.v_cache[layer])
        p.rope_cos, p.rope_sin = _ptr(bufs.rope_cos), _ptr(bufs.rope_sin)
        p.positions = _ptr(bufs.positions)
        p.partial = _ptr(bufs.partial)
        if getattr(bufs, "page_table", None) is not None:       # paged KV pools
            p.page_table = _ptr(bufs.page_table)
            p.max_pages = bufs.page_table.shape[1]
        if opts.prefill:
            if not attn_mma:
                raise ValueError("chunked prefill needs the tensor-core attention path")
            p.prefill = 1
        p.out = _ptr(out)
        p.M, p.ldqkv = B, spec.qkv_dim
        p.q_heads, p.kv_heads, p.head_dim = spec.q_heads, spec.kv_heads, hd
        p.group, p.kv_head = spec.group, h
        p.split, p.n_splits, p.t_max = bufs.split, bufs.n_splits, bufs.t_max
        p.eps, p.scale = spec.eps, hd ** -0.5
        # one item per unit (small batch): two warps share each (item, head)
        # and write two partial pieces; otherwise one warp per (item, head)
        if attn_mma:
            p.mma = 1
            # tensor-core path (csrc attn_mma_pass): warps per item so that
            # every consumer warp has work -- 8 / wpi items per pass, whose
            # 2 * 8 / wpi K/V slots must fit the 10-slot ring (wpi >= 2)
            p.sub_splits = int(os.environ.get("MK_ATTN_WPI", "1"))
        else:
            p.sub_splits = 2 if (B * bufs.n_splits <= u_attn and 8 % (2 * spec.group) == 0) else 1
        return blob.add(p)

    def gemm_tile_of(kind):
        for t in g.tasks:
            if t.op_kind is kind:
                return tuple(t.tile_shape)
        return None

    gu_fused = g.mode == "chiplet"
    attn_mma = (opts.attn_mma and hd == 128 and bufs.split == 64 and spec.group <= 4
                and B >= ATTN_MMA_MIN_BATCH)
    # barrier-free tensor-core attention merges the splits itself
    fused_reduce = (attn_mma and opts.fuse_attn_reduce
                    and int(os.environ.get("MK_ATTN_WPI", "1")) == 1)
    ksplit = opts.ksplit and per_die and bufs.kpart is not None
    # tcgen05 graphs: each RMSNorm folded into its consumer's weights
    # (runtime.build_state packs W * gamma); the residual-producing GEMMs
    # emit per-tile sums of squares, the consumer scales by 1/rms
    fold = (opts.fuse_norm and getattr(bufs, "fold_norm", False) and opts.tp_world == 1)
    fuse = not fold and opts.fuse_norm and all(
        stages(B, d, tl) and not is_umma_tile(tl, f)
        for tl, f in ((gemm_tile_of(OpKind.QKV_PROJ), False),
                      (gemm_tile_of(OpKind.GATE_UP_SILU), gu_fused),
                      (opts.lm_tile, False)))
    # attention units: at most one per worker (a second unit on a worker
    # would serialise behind the first)
    u_attn = max(1, total_workers // spec.kv_heads)
    u_rows = min(B, 16)
    silu_meta = _silu_meta(g, B, F)

    # event -> event its (no-op) signaller waited on: a fused RMSNorm task
    # without the L0 embedding gather does no work, so waiting on its event
    # would only add a completion hop to the critical path
    bypass = {}

    tp = opts.tp_world > 1
    if tp and (opts.tp_layout is None or opts.tp_layout.world != opts.tp_world):
        raise ValueError("tensor-parallel lowering needs the group's TPLayout")
    kv0 = opts.tp_rank * spec.kv_heads              # first kv head of this rank's shard
    # the last task of every (layer, row-parallel op): its allreduce follows it
    last_of = {}
    for gi, t in enumerate(g.tasks):
        if t.op_kind in (OpKind.O_PROJ_RESIDUAL, OpKind.DOWN_PROJ_RESIDUAL):
            last_of[(t.id.split(".")[0], t.op_kind)] = gi
    u_ar = max(1, min(total_workers, d // 8 // 32))

    def add_allreduce(layer, kind, wait, res, y):
        point = 2 * layer + (0 if kind is OpKind.O_PROJ_RESIDUAL else 1)
        ev = f"e.L{layer}.{'o' if point % 2 == 0 else 'down'}_allreduce"
        ev_index[ev] = len(event_names)
        event_names.append(ev)
        required.append(1)
        p = L.TPParams()
        p.recv_off = opts.tp_layout.recv_off(point)
        p.flag_off = opts.tp_layout.flag_off(point)
        p.res, p.y = _ptr(res), _ptr(y)
        p.M, p.d = B, d
        add_task(f"L{layer}.{'o' if point % 2 == 0 else 'down'}_allreduce.t0", -1,
                 L.OP_TP_ALLREDUCE, L.LEVEL_CU, None, wait, ev, blob.add(p), layer,
                 n_items=d // 8, n_units=u_ar)
        bypass[wait] = ev            # consumers of the partial GEMM wait on the sum

    for gi, t in enumerate(g.tasks):
        layer = int(t.id.split(".")[0][1:])
        lb = bufs.layers[layer]
        wl = bufs.w_layers[layer]
        wait = t.wait_events[0] if t.wait_events else None
        wait = bypass.get(wait, wait)
        level = {TaskLevel.CHIPLET: L.LEVEL_CHIPLET, TaskLevel.CU: L.LEVEL_CU,
                 TaskLevel.WAVEFRONT: L.LEVEL_WAVEFRONT}[t.level]
        op = t.op_kind
        if op is OpKind.RMS_NORM:
            first = t.id.endswith("rms1.t0")
            if first:
                src = bufs.x_in0 if layer == 0 else bufs.layers[layer - 1]["x_out"]
                po = norm_params(lb, src, wl["in_norm"], lb["normed1"],
                                 embed=(layer == 0), fused=fuse or fold,
                                 ss_out=bufs.ss_in0 if (fold and layer == 0) else None)
            else:
                po = norm_params(lb, lb["x_mid"], wl["post_norm"], lb["normed2"],
                                 fused=fuse or fold)
            add_task(t.id, gi, L.OP_RMSNORM, level, None, wait, t.signal_event,
                     po, layer, n_items=B, n_units=u_rows)
            if (fuse or fold) and opts.bypass_noop and not (first and layer == 0) and wait:
                bypass[t.signal_event] = wait
        elif op in (OpKind.QKV_PROJ, OpKind.O_PROJ_RESIDUAL,
                    OpKind.GATE_UP_SILU, OpKind.DOWN_PROJ_RESIDUAL):
            # this rank's shard of the device-wide GEMM (== the graph's
            # gemm_shape without tensor parallelism)
            M, K, N = {OpKind.QKV_PROJ: (B, d, spec.qkv_dim),
                       OpKind.O_PROJ_RESIDUAL: (B, spec.q_heads * hd, d),
                       OpKind.GATE_UP_SILU: (B, d, 2 * F),
                       OpKind.DOWN_PROJ_RESIDUAL: (B, F, d)}[op]
            if not tp:
                assert (M, K, N) == tuple(t.gemm_shape), (t.id, (M, K, N), t.gemm_shape)
            tile = tuple(t.tile_shape)
            x_in = bufs.x_in0 if layer == 0 else bufs.layers[layer - 1]["x_out"]
            gamma = None
            ss_in = ss_out = None
            n_parts = d // 32
            if op is OpKind.QKV_PROJ:
                w, x, y, res, epi, ldx, ldy = (bufs.w_packed[layer]["qkv"],
                                              lb["normed1"], lb["qkv_out"], None,
                                              L.EPI_NONE, d, spec.qkv_dim)
                if fuse:
                    x, gamma = x_in, wl["in_norm"]
                if fold:
                    x = x_in
                    ss_in = (bufs.ss_in0, 1) if layer == 0 else \
                        (bufs.layers[layer - 1]["ss_out"], n_parts)
            elif op is OpKind.O_PROJ_RESIDUAL:
                w, x, y, res, epi, ldx, ldy = (bufs.w_packed[layer]["o"],
                                              lb["attn_out"], lb["x_mid"], x_in,
                                              L.EPI_RESIDUAL, K, d)
                if fold:
                    ss_out = lb["ss_mid"]
            elif op is OpKind.GATE_UP_SILU:
                fused = t.level is TaskLevel.CHIPLET
                w = bufs.w_packed[layer]["gate_up"]
                x, ldx = lb["normed2"], d
                if fuse:
                    x, gamma = lb["x_mid"], wl["post_norm"]
                if fold:
                    x, ss_in = lb["x_mid"], (lb["ss_mid"], n_parts)
                if fused:
                    y, epi, ldy = lb["silu_out"], L.EPI_SILU, F
                else:
                    y, epi, ldy = lb["gu_out"], L.EPI_NONE, 2 * F
                res = None
            else:
                w, x, y, res, epi, ldx, ldy = (bufs.w_packed[layer]["down"],
                                              lb["silu_out"], lb["x_out"],
                                              lb["x_mid"], L.EPI_RESIDUAL, F, d)
                if fold:
                    ss_out = lb["ss_out"]
            ar = None
            if tp and op in (OpKind.O_PROJ_RESIDUAL, OpKind.DOWN_PROJ_RESIDUAL):
                # row-parallel: the fp32 partial goes to every rank (y is this
                # rank's slot offset in the exchange regions), residual later
                ar = (res, y)
                point = 2 * layer + (0 if op is OpKind.O_PROJ_RESIDUAL else 1)
                y = _Off(opts.tp_layout.slot_off(point, opts.tp_rank))
                res, epi = None, L.EPI_PARTIAL
            if t.level is TaskLevel.CHIPLET:
                X = g.machine.num_xcds
                n_loc = N // X
                xd = t.xcd_binding
                col0 = xd * (n_loc // 2 if epi == L.EPI_SILU else n_loc)
                po = gemm_params(_ptr(w, xd * n_loc * K), _ptr(x), _ptr(y),
                                 _ptr(res), M, K, n_loc, tile, ldx, ldy, d,
                                 col0, epi, xd, gamma=gamma, ksplit=ksplit,
                                 ss_in=ss_in, ss_out=ss_out)
                add_task(t.id, gi, L.OP_GEMM, level, xd, wait, t.signal_event,
                         po, layer, n_items=0)
            else:
                work = t.work
                po = gemm_params(_ptr(w), _ptr(x), _ptr(y), _ptr(res), M, K, N,
                                 tile, ldx, ldy, d, 0, epi, 0,
                                 tm=work.m_idx, tn=work.n_idx, gamma=gamma,
                                 ss_in=ss_in, ss_out=ss_out)
                add_task(t.id, gi, L.OP_GEMM, level, None, wait, t.signal_event,
                         po, layer)
            if ar is not None and gi == last_of[(t.id.split(".")[0], op)]:
                add_allreduce(layer, op, t.signal_event, *ar)
        elif op is OpKind.ATTN_PARTIAL:
            # tensor parallel: kv heads outside this rank's shard keep their
            # task (the graph topology is unchanged) with no items
            h = int(t.id.rsplit(".t", 1)[1]) - kv0
            mine = 0 <= h < spec.kv_heads
            po = attn_params(layer, h if mine else 0, out=lb["attn_out"], fuse=True)
            add_task(t.id, gi, L.OP_ATTN_PARTIAL, level, None, wait,
                     t.signal_event, po, layer, n_items=B * bufs.n_splits if mine else 0,
                     n_units=u_attn)
        elif op is OpKind.ATTN_REDUCE:
            h = int(t.id.rsplit(".t", 1)[1]) - kv0
            mine = 0 <= h < spec.kv_heads
            if not mine:
                po = attn_params(layer, 0, out=lb["attn_out"], reduce_noop=fused_reduce)
                add_task(t.id, gi, L.OP_ATTN_REDUCE, level, None, wait,
                         t.signal_event, po, layer, n_items=0, n_units=1)
                continue
            po = attn_params(layer, h, out=lb["attn_out"], reduce_noop=fused_reduce)
            if fused_reduce:
                # merged inside ATTN_PARTIAL: the task stays in the graph as a
                # no-op (one unit), its consumers wait on the partial stage's event
                bypass[t.signal_event] = wait
            add_task(t.id, gi, L.OP_ATTN_REDUCE, level, None, wait,
                     t.signal_event, po, layer, n_items=B,
                     n_units=1 if fused_reduce else u_attn)
        elif op is OpKind.SILU:
            row0, rows, col0, cols = silu_meta[t.id]
            p = L.SiluParams()
            p.gu, p.y = _ptr(lb["gu_out"]), _ptr(lb["silu_out"])
            p.F, p.row0, p.rows, p.col0, p.cols = F, row0, rows, col0, cols
            add_task(t.id, gi, L.OP_SILU, level, None, wait, t.signal_event,
                     blob.add(p), layer)
        else:
            raise ValueError(f"cannot lower {op}")

    # ---- appended stages: final norm -> LM head -> argmax ---------------
    last_event = bypass.get(g.tasks[-1].signal_event, g.tasks[-1].signal_event)
    n_layers = len(bufs.layers)
    for e in ("e.final_norm", "e.lm_head", "e.argmax"):
        ev_index[e] = len(event_names)
        event_names.append(e)
        required.append(0)
    x_last = bufs.layers[n_layers - 1]["x_out"]
    po = norm_params(None, x_last, bufs.final_norm, bufs.final_normed, fused=fuse or fold)
    lm_x = x_last if (fuse or fold) else bufs.final_normed
    lm_gamma = bufs.final_norm if fuse else None
    lm_ss = (bufs.layers[n_layers - 1]["ss_out"], d // 32) if fold else None
    add_task("final_norm.t0", -1, L.OP_RMSNORM, L.LEVEL_CU, None, last_event,
             "e.final_norm", po, n_layers, n_items=B, n_units=u_rows)
    lm_wait = last_event if ((fuse or fold) and opts.bypass_noop) else "e.final_norm"
    required[ev_index["e.final_norm"]] = 1
    t_m, t_n, t_k = opts.lm_tile
    V = bufs.vocab_pad or spec.vocab          # padded for 128-row tcgen05 tiles
    logits = bufs.logits
    if per_die:
        X = opts.n_dies
        n_loc = V // X
        for xd in range(X):
            po = gemm_params(_ptr(bufs.lm_packed, xd * n_loc * d),
                             _ptr(lm_x), _ptr(logits), None,
                             B, d, n_loc, (t_m, t_n, t_k), d, V, d,
                             xd * n_loc, L.EPI_LOGITS, xd,
                             amax_base=xd * opts.workers, gamma=lm_gamma,
                             y_cols=spec.vocab, ksplit=ksplit, ss_in=lm_ss)
            add_task(f"lm_head.x{xd}", -1, L.OP_GEMM, L.LEVEL_CHIPLET, xd,
                     lm_wait, "e.lm_head", po, n_layers, n_items=0)
        required[ev_index["e.lm_head"]] = X
        amax_slots = X * opts.workers
    else:
        mt, nt = _cdiv(B, t_m), V // t_n
        for m in range(mt):
            for n in range(nt):
                po = gemm_params(_ptr(bufs.lm_packed), _ptr(lm_x),
                                 _ptr(logits), None, B, d, V, (t_m, t_n, t_k),
                                 d, V, d, 0, L.EPI_LOGITS, 0, tm=m, tn=n,
                                 amax_base=n, gamma=lm_gamma, y_cols=spec.vocab,
                                 ss_in=lm_ss)
                add_task(f"lm_head.t{m * nt + n}", -1, L.OP_GEMM, L.LEVEL_CU,
                         None, lm_wait, "e.lm_head", po, n_layers)
        required[ev_index["e.lm_head"]] = mt * nt
        amax_slots = nt
    if tp:
        # vocab-parallel LM head: (max, global index) of the shard to every
        # rank, the same global pick on each (lowest index on ties)
        p = L.TPParams()
        p.flag_off = opts.tp_layout.flag_off(opts.tp_layout.argmax_point)
        p.gather_off = opts.tp_layout.gather_off
        p.amax_val, p.amax_idx = _ptr(bufs.amax_val), _ptr(bufs.amax_idx)
        p.out_tokens, p.next_tokens = _ptr(bufs.out_tokens), _ptr(bufs.tokens)
        p.positions = _ptr(bufs.positions)
        p.M, p.d, p.n_slots, p.vocab0 = B, d, amax_slots, opts.tp_rank * spec.vocab
        add_task("argmax.t0", -1, L.OP_TP_ARGMAX, L.LEVEL_CU, None, "e.lm_head",
                 "e.argmax", blob.add(p), n_layers, n_items=B, n_units=1)
    else:
        p = L.ArgmaxParams()
        p.amax_val, p.amax_idx = _ptr(bufs.amax_val), _ptr(bufs.amax_idx)
        p.out_tokens, p.next_tokens = _ptr(bufs.out_tokens), _ptr(bufs.tokens)
        p.positions = _ptr(bufs.positions)
        p.M, p.n_slots = B, amax_slots
        add_task("argmax.t0", -1, L.OP_ARGMAX, L.LEVEL_CU, None, "e.lm_head",
                 "e.argmax", blob.add(p), n_layers, n_items=B, n_units=u_rows)
    required[ev_index["e.argmax"]] = 1

    flat_units = [u for s in units_by_sched for u in s]
    begin = [0]
    for s in units_by_sched:
        begin.append(begin[-1] + len(s))
    t_arr = (L.Task * len(tasks))(*tasks)
    u_arr = (L.Unit * len(flat_units))(
        *[L.Unit(ti, ib, ie, 0) for ti, ib, ie in flat_units])
    b_arr = (C.c_int32 * len(begin))(*begin)
    r_arr = (C.c_int32 * len(required))(*required)
    return Lowered(t_arr, u_arr, b_arr, r_arr, bytes(blob.data), event_names,
                   names, gidx, n_sub[0], n_sched, opts.sched_mode,
                   opts.workers, amax_slots, kv_swizzled=attn_mma,
                   positions=_ptr(bufs.positions) or 0, n_rows=B,
                   tokens=_ptr(bufs.tokens) or 0, out_tokens=_ptr(bufs.out_tokens) or 0)


def _silu_meta(g: TaskGraph, B: int, F: int):
    """(row0, rows, col0, cols) of every standard-mode SiLU task
    (ref taskgraph.py:476-504: ids t{group*n_chunks + chunk})."""
    out = {}
    by_layer = {}
    for t in g.tasks:
        if t.op_kind is OpKind.SILU:
            by_layer.setdefault(t.id.split(".")[0], []).append(t)
    for tasks in by_layer.values():
        gu = [t for t in g.tasks if t.op_kind is OpKind.GATE_UP_SILU][0]
        t_m = gu.tile_shape[0]
        groups = _cdiv(B, t_m)
        n_chunks = len(tasks) // groups
        dt = 2
        first_rows = min(t_m, B)
        chunk = tasks[0].work.reads[0][1] // (first_rows * dt)
        for t in tasks:
            k = int(t.id.rsplit(".t", 1)[1])
            grp, j = divmod(k, n_chunks)
            rows = min(t_m, B - grp * t_m)
            cols = min(chunk, F - j * chunk)
            out[t.id] = (grp * t_m, rows, j * chunk, cols)
    return out
