"""Host graph compiler invariants (CPU only: descriptors are lowered against
CPU tensors, nothing is launched)."""

import pytest

from paper_2604_15379_b200 import (Distribution, Traversal, build_decoder_layer,
                                   model_preset, preset)
from paper_2604_15379_b200 import _lib as L
from paper_2604_15379_b200.analytics import device_tiles
from paper_2604_15379_b200.lowering import LoweringOptions, lower
from paper_2604_15379_b200.runtime import _default_lm_tile, build_state
from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights

W = 73


def _lower(mode, B, fanout=True, bypass=True, layers=2, per_die=None):
    m = model_preset("toy")
    mach = preset("b200")
    g = build_decoder_layer(m, mach, mode, B, tile_overrides=device_tiles(m, mach, mode, B),
                            layers=layers)
    spec = Qwen3Spec.toy(layers=layers)
    w = Qwen3Weights.random(spec, seed=1)
    per_die = (mode == "chiplet") if per_die is None else per_die
    lm = _default_lm_tile(spec, B)
    slots = 2 * W if per_die else spec.vocab // lm[1]
    st = build_state(g, w, 128, lm, slots, device="cpu")
    opts = LoweringOptions(sched_mode=L.SCHED_PER_DIE if per_die else L.SCHED_FLAT,
                           workers=W if per_die else 147, n_dies=2, fanout=fanout,
                           lm_tile=lm, bypass_noop=bypass)
    return g, lower(g, spec, st, opts)


@pytest.mark.parametrize("mode", ["chiplet", "standard"])
@pytest.mark.parametrize("B", [1, 5, 20])
@pytest.mark.parametrize("fanout", [True, False])
def test_descriptors_cover_graph(mode, B, fanout):
    g, low = _lower(mode, B, fanout=fanout)
    tasks = [low.tasks[i] for i in range(len(low.tasks))]
    # every graph task lowered exactly once, in graph order, + 3 head tasks
    gidx = [t.graph_index for t in tasks if t.graph_index >= 0]
    assert gidx == list(range(len(g.tasks)))
    assert low.task_names[:len(g.tasks)] == [t.id for t in g.tasks]
    assert [n.split(".")[0] for n in low.task_names[len(g.tasks):]][:1] == ["final_norm"]
    # event required counts == number of device tasks signalling each event
    sig = {}
    for t in tasks:
        sig[t.signal] = sig.get(t.signal, 0) + 1
    for e, name in enumerate(low.event_names):
        assert low.event_required[e] == sig.get(e, 0), name
    # graph events keep the reference required_count
    for e, name in enumerate(low.event_names[:len(g.events)]):
        assert low.event_required[e] == g.events[name].required_count
    # units: each CU task's items covered exactly once, die tasks once per die list
    units = [low.units[i] for i in range(len(low.units))]
    cover = {}
    for u in units:
        cover.setdefault(u.task, []).append((u.item_begin, u.item_end))
    for ti, t in enumerate(tasks):
        spans = sorted(cover[ti])
        assert len(spans) == (1 if t.level == L.LEVEL_CHIPLET else t.n_units)
        if t.level != L.LEVEL_CHIPLET:
            assert spans[0][0] == 0 and spans[-1][1] == t.n_items
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
        assert (t.sub_ctr >= 0) == (t.n_units > 1)
    # scheduler lists: die tasks in their die's list
    begin = list(low.sched_begin)
    for s in range(low.n_sched):
        for u in units[begin[s]:begin[s + 1]]:
            t = tasks[u.task]
            if t.level == L.LEVEL_CHIPLET and low.n_sched > 1:
                assert t.die == s


def test_fanout_off_means_one_unit_per_task():
    g, low = _lower("chiplet", 4, fanout=False)
    assert len(low.units) == len(low.tasks)


def test_bypass_redirects_only_fused_norm_consumers():
    g, on = _lower("chiplet", 1, bypass=True)
    _, off = _lower("chiplet", 1, bypass=False)
    ev = on.event_names
    changed = []
    for i in range(len(on.tasks)):
        a, b = on.tasks[i], off.tasks[i]
        assert a.signal == b.signal
        if a.wait0 != b.wait0:
            changed.append((on.task_names[i], ev[b.wait0], ev[a.wait0]))
    # L1.qkv skips L1.rms1 (no-op), gate_up skips rms2, lm_head skips final_norm;
    # L0.qkv still waits on L0.rms1 (embedding gather)
    names = {c[0].rsplit(".", 1)[0] for c in changed}
    assert "L0.qkv" not in names
    assert {"L1.qkv", "L0.gate_up", "L1.gate_up", "lm_head"} <= names
    for name, old, new in changed:
        assert "rms" in old or "final_norm" in old


def test_flat_scheduler_rejects_die_bound_graph():
    with pytest.raises(ValueError, match="die-unaware"):
        _lower("chiplet", 1, per_die=False)


def test_gemm_params_die_slabs():
    g, low = _lower("chiplet", 2, layers=1)
    import ctypes
    blob = low.params
    for i in range(len(low.tasks)):
        t = low.tasks[i]
        if t.op != L.OP_GEMM or t.level != L.LEVEL_CHIPLET or t.graph_index < 0:
            continue
        p = L.GemmParams.from_buffer_copy(blob[t.param_off:t.param_off + ctypes.sizeof(L.GemmParams)])
        gt = g.tasks[t.graph_index]
        n_loc = gt.gemm_shape[2] // 2
        assert p.N == n_loc and p.xcd == gt.xcd_binding
        width = n_loc // 2 if p.epilogue == L.EPI_SILU else n_loc
        assert p.y_col0 == gt.xcd_binding * width


def _owner(s, S, W):
    """Inverse of the K-split range starts w*S/W (csrc range_owner)."""
    return ((s + 1) * W + S - 1) // S - 1


def test_ksplit_ranges_cover_every_slot_once_and_pieces_are_consistent():
    """Host restatement of the device K-split partition (csrc RangeIter /
    tile_pieces): worker ranges tile the slot sequence exactly once, the
    owner formula inverts the range starts, and the pieces of every cut tile
    are the non-empty ranges between the owners of its first and last slot
    (also when there are more workers than slots)."""
    for tiles, chunks, W in [(24, 64, 71), (16, 192, 71), (96, 64, 69), (2, 1, 71),
                             (32, 2, 71), (594, 64, 74), (5, 3, 7)]:
        S = tiles * chunks
        starts = [S * w // W for w in range(W + 1)]
        seen = [0] * S
        for w in range(W):
            for s in range(starts[w], starts[w + 1]):
                seen[s] += 1
                assert _owner(s, S, W) == w
        assert seen == [1] * S
        for t in range(tiles):
            a, b = t * chunks, t * chunks + chunks - 1
            fw, lw = _owner(a, S, W), _owner(b, S, W)
            pieces = [w for w in range(fw, lw + 1) if starts[w] != starts[w + 1]]
            covering = sorted({_owner(s, S, W) for s in range(a, b + 1)})
            assert pieces == covering


def test_ksplit_pays_only_for_unbalanced_whole_tile_ownership():
    from paper_2604_15379_b200.lowering import gemv_fast_shape, ksplit_pays
    assert not ksplit_pays(384, 71)      # B=1 qkv GEMV tiles: 6 rounds, 90% balance
    assert ksplit_pays(16, 71)           # tcgen05 o_proj / down: 16 tiles, 71 workers
    assert ksplit_pays(96, 71)           # tcgen05 gate_up: 2 rounds, 68% balance
    assert not ksplit_pays(142, 71)      # exactly two rounds
    assert gemv_fast_shape(1, 8, 1024) and gemv_fast_shape(8, 32, 256)
    assert not gemv_fast_shape(16, 32, 256)


def _lower_mini(B, **kw):
    """Qwen3-shaped mini model (head_dim 128): the tensor-core attention path."""
    from paper_2604_15379_b200.machine import ModelConfig
    m = ModelConfig(hidden_dim=512, ffn_dim=1024, num_layers=2, q_heads=4, kv_heads=2,
                    dtype_bytes=2)
    mach = preset("b200")
    g = build_decoder_layer(m, mach, "chiplet", B, tile_overrides=device_tiles(m, mach, "chiplet", B),
                            layers=2)
    spec = Qwen3Spec(512, 1024, 2, 4, 2, 128, 1024)
    w = Qwen3Weights.random(spec, seed=2)
    lm = _default_lm_tile(spec, B)
    st = build_state(g, w, 128, lm, 2 * W, device="cpu")
    opts = LoweringOptions(sched_mode=L.SCHED_PER_DIE, workers=W, n_dies=2, lm_tile=lm, **kw)
    return g, lower(g, spec, st, opts)


def _params(low, t, cls):
    import ctypes
    return cls.from_buffer_copy(low.params[t.param_off:t.param_off + ctypes.sizeof(cls)])


@pytest.mark.parametrize("fuse", [False, True])
def test_tensor_core_attention_lowering(fuse):
    """head_dim 128: ATTN_PARTIAL on the tensor-core path (one warp per item);
    with the fused split merge every row gets an arrival counter, ATTN_REDUCE
    becomes a one-unit no-op and its consumers wait on the partial stage."""
    g, low = _lower_mini(16, fuse_attn_reduce=fuse)
    tasks = [low.tasks[i] for i in range(len(low.tasks))]
    names = low.task_names
    ctrs = []
    for t in tasks:
        if t.op == L.OP_ATTN_PARTIAL:
            p = _params(low, t, L.AttnParams)
            assert p.mma == 1 and p.sub_splits == 1 and p.t_max % 64 == 0
            assert p.fuse_reduce == (1 if fuse else 0)
            if fuse:
                ctrs.append(p.red_ctr0)
        if t.op == L.OP_ATTN_REDUCE:
            assert _params(low, t, L.AttnParams).fuse_reduce == (1 if fuse else 0)
            assert (t.n_units == 1) == fuse
    if fuse:   # disjoint per-row counters in the sub-counter space
        assert len(set(ctrs)) == len(ctrs) and max(ctrs) + 16 <= low.n_sub
    ev = {n: i for i, n in enumerate(low.event_names)}
    o_proj = [t for t, n in zip(tasks, names) if ".o_proj." in n]
    want = "attn_partial" if fuse else "attn_reduce"
    for t in o_proj:
        assert low.event_names[t.wait0].endswith(want), low.event_names[t.wait0]
    assert ev  # events lowered


def _ref_chipletsim():
    import os
    import sys
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference package not present (build container only)")
    if src not in sys.path:
        sys.path.insert(0, src)
    return pytest.importorskip("chipletsim")


@pytest.mark.parametrize("mode", ["chiplet", "standard"])
@pytest.mark.parametrize("B", [1, 8])
def test_lowers_a_graph_built_by_the_reference(mode, B):
    """Drop-in boundary: a TaskGraph built by the REFERENCE's own
    build_decoder_layer (chipletsim, ref taskgraph.py:355-526) lowers to
    exactly the device descriptors of the same graph built here."""
    import os

    _ref_chipletsim()
    from chipletsim import machine as rm
    from chipletsim import taskgraph as rt
    gold = os.path.join(os.path.dirname(__file__), "golden", "b200_machine.json")
    m, mach = model_preset("toy"), preset("b200")
    tiles = device_tiles(m, mach, mode, B)
    rtiles = {(k if k == "silu_chunk" else rt.OpKind(k.value)): v for k, v in tiles.items()}
    g_ref = rt.build_decoder_layer(rm.model_preset("toy"), rm.load_machine(gold), mode, B,
                                   tile_overrides=rtiles, layers=2)
    g_own = build_decoder_layer(m, mach, mode, B, tile_overrides=tiles, layers=2)
    spec = Qwen3Spec.toy(layers=2)
    w = Qwen3Weights.random(spec, seed=1)
    lm = _default_lm_tile(spec, B)
    per_die = mode == "chiplet"
    slots = 2 * W if per_die else spec.vocab // lm[1]
    opts = LoweringOptions(sched_mode=L.SCHED_PER_DIE if per_die else L.SCHED_FLAT,
                           workers=W if per_die else 147, n_dies=2, fanout=True, lm_tile=lm)
    lows = []
    for g in (g_ref, g_own):
        st = build_state(g, w, 128, lm, slots, device="cpu")
        lows.append(lower(g, spec, st, opts))
    a, b = lows
    assert a.task_names == b.task_names and a.event_names == b.event_names
    assert list(a.event_required) == list(b.event_required)
    assert bytes(a.tasks) == bytes(b.tasks) and bytes(a.units) == bytes(b.units)
    assert list(a.sched_begin) == list(b.sched_begin)
