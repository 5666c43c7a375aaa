"""Pin the sync-accounting restatement (oracle/sched_accounting.py) against
the reference simulator's own counters (tests/golden/sim_counters.json)."""

import json
import os

import pytest

from oracle.cases import TILE_SPECS
from oracle.sched_accounting import dispatch_partition, expected_counters
from paper_2604_15379_b200 import (OpKind, build_decoder_layer, build_gemm_graph,
                                   load_machine, model_preset, preset)
from paper_2604_15379_b200.analytics import fit_tiles

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SIMS = json.load(open(os.path.join(GOLD, "sim_counters.json")))


def _machine(name):
    if name == "b200":
        return load_machine(os.path.join(GOLD, "b200_machine.json"))
    return preset(name)


def _graph(c):
    mach = _machine(c["machine"])
    if c["kind"] == "gemm":
        return mach, build_gemm_graph(mach, tuple(c["shape"]), tuple(c["tiles"]),
                                      c["mode"])
    model = model_preset(c["model"])
    if c["tiles"] == "fit":
        tiles = fit_tiles(model, mach, c["mode"])
    else:
        raw = TILE_SPECS[c["tiles"]]
        tiles = {(k if k == "silu_chunk" else OpKind(k)):
                 (v if k == "silu_chunk" else tuple(v)) for k, v in raw.items()}
    return mach, build_decoder_layer(model, mach, c["mode"], c["batch"],
                                     tile_overrides=tiles, layers=c["layers"])


@pytest.mark.parametrize("case", SIMS, ids=lambda c: f"{c['kind']}-{c['machine']}-{c['mode']}")
def test_counters_match_reference_simulate(case):
    mach, g = _graph(case)
    exp = expected_counters(g, mach.workers_per_xcd)
    for k in ("dispatches", "fences", "local_atomics", "global_atomics"):
        assert exp[k] == case[k], k


@pytest.mark.parametrize("case", [c for c in SIMS if c.get("log")],
                         ids=lambda c: f"{c['machine']}-{c['mode']}-b{c['batch']}")
def test_per_die_dispatch_order_matches_reference_log(case):
    mach, g = _graph(case)
    lists = dispatch_partition(g, mach.num_xcds)
    per_die = [[] for _ in range(mach.num_xcds)]
    for step, actor, action, tid in case["log"]:
        if action == "dispatch":
            per_die[int(actor.split(".x")[1])].append(tid)
    assert per_die == lists


SIMS_W = json.load(open(os.path.join(GOLD, "sim_counters_w.json")))


@pytest.mark.parametrize("case", SIMS_W, ids=lambda c: f"W{c['workers']}-{c['model']}")
def test_counters_match_reference_simulate_any_w(case):
    """The restatement at every workers-per-die W a probed B200 can give
    (fixture: ref simulate() at W = 64..77, oracle/gen_sim_w.py)."""
    from dataclasses import replace
    from paper_2604_15379_b200.analytics import device_tiles
    W = case["workers"]
    base = load_machine(os.path.join(GOLD, "b200_machine.json"))
    mach = replace(base, cus_per_xcd=W + 1, workers_per_xcd=W)
    model = model_preset(case["model"])
    tiles = (fit_tiles(model, mach, "chiplet") if case["tiles"] == "fit"
             else device_tiles(model, mach, "chiplet", case["batch"]))
    g = build_decoder_layer(model, mach, "chiplet", case["batch"], tile_overrides=tiles,
                            layers=case["layers"])
    exp = expected_counters(g, W)
    for k in ("dispatches", "fences", "local_atomics", "global_atomics"):
        assert exp[k] == case[k], k
    # linear in layers: the 36-layer device check scales the same formula
    g36 = build_decoder_layer(model, mach, "chiplet", case["batch"], tile_overrides=tiles,
                              layers=case["layers"] * 3)
    e36 = expected_counters(g36, W)
    assert all(e36[k] == 3 * exp[k] for k in exp)
