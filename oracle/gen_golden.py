"""Generate golden fixtures from the REFERENCE itself (test infrastructure).

Run in the build container, where ``/root/reference`` exists:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python oracle/gen_golden.py

It imports the reference package ``chipletsim`` and writes, under
``tests/golden/``:

* ``b200_machine.json`` -- the 2-die B200 machine config fed to both builders;
* ``graphs.json`` -- for every (machine, model, mode, batch, layers, tiles)
  case: task/event counts and the sha256 of ``json.dumps(graph_to_json(g))``
  (ref taskgraph.py:647-682), plus the full JSON for the small toy cases;
* ``schedules.json`` -- ``schedule_to_json`` (ref traversal.py:342-354) over a
  grid of partitions / worker counts / traversals / distributions;
* ``sim_counters.json`` -- ``simulate`` (ref runtime.py:253-548) sync
  accounting (dispatches, fences, global and local atomics) and the event-log
  dispatch/complete order for small graphs; the device scheduler's counters
  are checked against these numbers.

The reference never runs on the GPU box; only these fixtures travel.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import chipletsim as ref  # noqa: E402  (reference, via PYTHONPATH)
from chipletsim import machine as ref_machine
from chipletsim import scenario as ref_scenario
from chipletsim import taskgraph as ref_tg
from chipletsim import traversal as ref_tr

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
from oracle.cases import (B200_MACHINE_JSON, GRAPH_CASES,  # noqa: E402
                          SCHEDULE_CASES, SIM_CASES, tiles_for)


def digest(doc) -> str:
    return hashlib.sha256(json.dumps(doc).encode()).hexdigest()


def ref_tiles(spec, model, machine, graph_mode):
    """Resolve a tile spec against the REFERENCE enums."""
    if spec == "fit":
        return ref_scenario.fit_tiles(model, machine, graph_mode)
    raw = tiles_for(spec)
    if raw is None:
        return None
    out = {}
    for k, v in raw.items():
        out[k if k == "silu_chunk" else ref_tg.OpKind(k)] = v
    return out


def machine_of(name):
    if name == "b200":
        return ref_machine.load_machine(OUT / "b200_machine.json")
    return ref_machine.preset(name)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / "b200_machine.json").write_text(
        json.dumps(B200_MACHINE_JSON, indent=1) + "\n")

    graphs = []
    for case in GRAPH_CASES:
        mach = machine_of(case["machine"])
        model = ref_machine.model_preset(case["model"])
        tiles = ref_tiles(case["tiles"], model, mach, case["mode"])
        g = ref_tg.build_decoder_layer(model, mach, case["mode"],
                                       case["batch"], tile_overrides=tiles,
                                       layers=case["layers"])
        ref_tg.validate_graph(g)
        doc = ref_tg.graph_to_json(g)
        rec = dict(case)
        rec.update(n_tasks=len(g.tasks), n_events=len(g.events),
                   op_counts=[list(map(list, c)) for c in g.op_counts],
                   sha256=digest(doc), notes=list(g.notes),
                   dot_sha256=hashlib.sha256(
                       ref_tg.graph_to_dot(g).encode()).hexdigest())
        if case.get("full"):
            rec["json"] = doc
        graphs.append(rec)
        print("graph", case["machine"], case["model"], case["mode"],
              case["batch"], case["layers"], case["tiles"], len(g.tasks))
    # gemm graphs (ref taskgraph.py:529-552)
    gemms = []
    for mname, shape, tiles, mode in [
            ("mi350", (1, 512, 3968), (16, 16, 256), "standard"),
            ("mi350", (1, 512, 3968), (16, 16, 256), "chiplet"),
            ("toy", (1, 64, 96), (16, 16, 64), "standard"),
            ("toy", (1, 64, 96), (16, 16, 64), "chiplet"),
            ("b200", (64, 4096, 6144), (16, 8, 1024), "chiplet"),
            ("b200", (64, 4096, 6144), (16, 8, 1024), "standard")]:
        g = ref_tg.build_gemm_graph(machine_of(mname), shape, tiles, mode)
        gemms.append(dict(machine=mname, shape=list(shape), tiles=list(tiles),
                          mode=mode, n_tasks=len(g.tasks),
                          sha256=digest(ref_tg.graph_to_json(g))))
    (OUT / "graphs.json").write_text(json.dumps(
        {"graphs": graphs, "gemm_graphs": gemms}, indent=0) + "\n")

    scheds = []
    for c in SCHEDULE_CASES:
        p = ref_tr.GemmPartition(
            M=c["m_tiles"] * 16, K=512, N_local=c["n_tiles"] * 8, T_M=16,
            T_N=8, T_K=256, weight_base=0, act_base=1 << 24,
            out_base=1 << 25, dtype_bytes=2)
        s = ref_tr.schedule(p, c["workers"], ref_tr.Traversal(c["traversal"]),
                            ref_tr.Distribution(c["distribution"]),
                            xcd=c["xcd"], num_xcds=c["num_xcds"],
                            window=c["window"])
        doc = ref_tr.schedule_to_json(s)
        rec = dict(c)
        rec["sha256"] = digest(doc)
        if c["m_tiles"] * c["n_tiles"] <= 64:
            rec["json"] = doc
        scheds.append(rec)
    (OUT / "schedules.json").write_text(json.dumps(scheds, indent=0) + "\n")

    sims = []
    for c in SIM_CASES:
        mach = machine_of(c["machine"])
        if c["kind"] == "layer":
            model = ref_machine.model_preset(c["model"])
            tiles = ref_tiles(c["tiles"], model, mach, c["mode"])
            g = ref_tg.build_decoder_layer(model, mach, c["mode"], c["batch"],
                                           tile_overrides=tiles,
                                           layers=c["layers"])
        else:
            g = ref_tg.build_gemm_graph(mach, tuple(c["shape"]),
                                        tuple(c["tiles"]), c["mode"])
        tr = ref.simulate(g, mach, traversal=ref_tr.Traversal(c["traversal"]),
                          distribution=ref_tr.Distribution(c["distribution"]))
        rec = dict(c)
        rec.update(dispatches=tr.dispatches, fences=tr.fences_issued,
                   global_atomics=tr.global_atomics,
                   local_atomics=tr.local_atomics, polls=tr.poll_count,
                   steps=tr.steps,
                   log=[list(e) for e in tr.event_log] if c.get("log") else None)
        sims.append(rec)
        print("sim", c)
    (OUT / "sim_counters.json").write_text(json.dumps(sims, indent=0) + "\n")


if __name__ == "__main__":
    main()
