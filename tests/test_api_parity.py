"""Drop-in API parity: our graph builder / schedules vs fixtures made by the reference.

Fixtures come from ``oracle/gen_golden.py`` (which imports the reference
``chipletsim`` in the build container).  Parity means byte-identical
``json.dumps(graph_to_json(g))`` (ref taskgraph.py:647-682) and
``schedule_to_json`` (ref traversal.py:342-354).
"""

import hashlib
import json
import os

import pytest

from oracle.cases import TILE_SPECS
from paper_2604_15379_b200 import (Distribution, GemmPartition, OpKind,
                                   Traversal, build_decoder_layer,
                                   build_gemm_graph, graph_to_dot,
                                   graph_to_json, load_machine, model_preset,
                                   preset, schedule, schedule_to_json,
                                   validate_graph)
from paper_2604_15379_b200.analytics import fit_tiles

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


GRAPHS = _load("graphs.json")
SCHEDS = _load("schedules.json")


def machine_of(name):
    if name == "b200":
        return load_machine(os.path.join(GOLD, "b200_machine.json"))
    return preset(name)


def tiles_of(spec, model, mach, mode):
    if spec == "fit":
        return fit_tiles(model, mach, mode)
    raw = TILE_SPECS[spec]
    if raw is None:
        return None
    return {(k if k == "silu_chunk" else OpKind(k)):
            (v if k == "silu_chunk" else tuple(v)) for k, v in raw.items()}


def sha(doc):
    return hashlib.sha256(json.dumps(doc).encode()).hexdigest()


def _case_id(c):
    return (f"{c['machine']}-{c['model']}-{c['mode']}-b{c['batch']}"
            f"-l{c['layers']}-{c['tiles']}")


@pytest.mark.parametrize("case", GRAPHS["graphs"], ids=_case_id)
def test_graph_json_matches_reference(case):
    mach = machine_of(case["machine"])
    model = model_preset(case["model"])
    g = build_decoder_layer(model, mach, case["mode"], case["batch"],
                            tile_overrides=tiles_of(case["tiles"], model, mach,
                                                    case["mode"]),
                            layers=case["layers"])
    validate_graph(g)
    assert len(g.tasks) == case["n_tasks"]
    assert len(g.events) == case["n_events"]
    assert [list(map(list, c)) for c in g.op_counts] == case["op_counts"]
    assert list(g.notes) == case["notes"]
    doc = graph_to_json(g)
    if "json" in case:
        assert doc == case["json"]
    assert sha(doc) == case["sha256"]
    assert hashlib.sha256(graph_to_dot(g).encode()).hexdigest() == \
        case["dot_sha256"]


@pytest.mark.parametrize("case", GRAPHS["gemm_graphs"],
                         ids=lambda c: f"{c['machine']}-{c['mode']}-{c['shape']}")
def test_gemm_graph_matches_reference(case):
    g = build_gemm_graph(machine_of(case["machine"]), tuple(case["shape"]),
                         tuple(case["tiles"]), case["mode"])
    assert len(g.tasks) == case["n_tasks"]
    assert sha(graph_to_json(g)) == case["sha256"]


def test_schedules_match_reference():
    for c in SCHEDS:
        p = GemmPartition(M=c["m_tiles"] * 16, K=512, N_local=c["n_tiles"] * 8,
                          T_M=16, T_N=8, T_K=256, weight_base=0,
                          act_base=1 << 24, out_base=1 << 25, dtype_bytes=2)
        s = schedule(p, c["workers"], Traversal(c["traversal"]),
                     Distribution(c["distribution"]), xcd=c["xcd"],
                     num_xcds=c["num_xcds"], window=c["window"])
        doc = schedule_to_json(s)
        if "json" in c:
            assert doc == c["json"], c
        assert sha(doc) == c["sha256"], c


PAYLOADS = _load("payloads.json")


@pytest.mark.parametrize("case", PAYLOADS, ids=lambda c: f"{c['machine']}-{c['model']}-{c['mode']}-b{c['batch']}")
def test_payloads_and_flops_match_reference(case):
    """Work payloads, per-task flops and stage flops -- the graph content
    graph_to_json omits -- equal the reference's (oracle/gen_extra_golden.py)."""
    from oracle.gen_extra_golden_doc import digest, payload_doc
    g = build_decoder_layer(model_preset(case["model"]), machine_of(case["machine"]),
                            case["mode"], case["batch"], layers=case["layers"])
    assert len(g.tasks) == case["n_tasks"]
    assert digest(payload_doc(g)) == case["sha256"]


def test_graph_error_messages_match_reference():
    """Every GraphError path of validate_graph / build_decoder_layer raises
    the reference's message (ref taskgraph.py:371-378, 555-612)."""
    from oracle.graph_mutations import BUILD_ERRORS, MUTATIONS
    from paper_2604_15379_b200 import GraphError
    want = _load("graph_errors.json")
    mach = preset("toy")
    base = build_decoder_layer(model_preset("toy"), mach, "chiplet", 2, layers=2)
    validate_graph(base)
    for name, fn in MUTATIONS.items():
        with pytest.raises(GraphError) as ei:
            validate_graph(fn(base))
        assert str(ei.value) == want[name], name
    for name, kw in BUILD_ERRORS.items():
        with pytest.raises(GraphError) as ei:
            build_decoder_layer(model_preset("toy"), mach, kw["mode"], kw["batch"],
                                layers=kw["layers"])
        assert str(ei.value) == want[name], name
