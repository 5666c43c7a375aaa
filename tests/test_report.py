"""Device-run records in the reference's report formats (report.py).

The fixture tests/golden/reports.json holds the REFERENCE's own
``SimTrace.to_json()`` / ``csv_row()`` / ``compare()`` /
``comparison_table`` / ``comparison_json`` output for toy-layer simulations
(oracle/gen_report_golden.py) and the metric numbers behind them; device
traces carrying the same numbers must produce identical records and text.
"""

import json
import math
import os

import pytest

from paper_2604_15379_b200 import report
from paper_2604_15379_b200.runtime import DeviceTrace

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return json.load(open(os.path.join(GOLD, "reports.json")))


def _trace(rec):
    j, n = rec["to_json"], rec["numbers"]
    met = report.DeviceMetrics(
        l2_hits=tuple(n["l2_hits"]), l2_misses=tuple(n["l2_misses"]),
        hbm_read_bytes_by_role=tuple(n["hbm_read_bytes_by_role"]),
        hbm_write_bytes_by_role=tuple(n["hbm_write_bytes_by_role"]),
        llc_hits=tuple(j["llc_hits"]), llc_misses=tuple(j["llc_misses"]),
        weight_rate=n["weight_l2_hit_rate"], source="fixture")
    return DeviceTrace(j["mode"], j["batch"], j["traversal"], j["distribution"], j["steps"],
                       j["fences"], j["global_atomics"], j["local_atomics"], j["polls"],
                       j["dispatches"], {}, (), metrics=met,
                       stage_costs=tuple(report.StageCost(**s) for s in j["stages"]),
                       estimated_time_s=j["estimated_time_s"], policy_notes=tuple(j["policy"]),
                       model_fingerprint=("toy",), fence_flush_lines=j["fence_flush_lines"])


def test_csv_columns_match_reference(gold):
    assert list(report.CSV_COLUMNS) == gold["csv_columns"]


def test_to_json_and_csv_row_match_reference(gold):
    for sid, rec in gold["traces"].items():
        tr = _trace(rec)
        assert tr.to_json() == rec["to_json"], sid
        assert tr.csv_row(sid) == rec["csv_row"], sid


def test_comparison_table_json_and_compare_match_reference(gold):
    rows = []
    for batch in (1, 8):
        rows.append((batch, {m: _trace(gold["traces"][f"{m}_b{batch}"])
                             for m in ("standard", "chiplet")}))
    assert report.comparison_table(rows) == gold["comparison_table"]
    assert json.loads(json.dumps(report.comparison_json(rows))) == gold["comparison_json"]
    c = report.compare(rows[1][1]["standard"], rows[1][1]["chiplet"]).to_json()
    assert c == gold["compare"]


def test_metrics_from_ncu_capture():
    """A real ncu --csv capture of one B=1 megakernel launch (r02, L2 prefetch
    on): its DRAM bytes and L2 sector hit rate become the trace metrics."""
    text = open(os.path.join(GOLD, "ncu_b1_metrics.csv")).read()
    m = report.metrics_from_ncu(text)
    assert m.source == "ncu"
    assert m.hbm_read_bytes == 15301553664
    assert abs(m.l2_hit_rate - 0.3172) < 1e-6
    with pytest.raises(ValueError):
        report.metrics_from_ncu(text, kernel="no_such_kernel")


def test_algorithmic_metrics_and_stage_costs_qwen3_8b():
    """Without a capture the step's algorithmic bytes stand in (L2 hit rate
    NaN); they equal analytics.decode_step_bytes, the bench's roofline bytes."""
    from paper_2604_15379_b200 import b200_from_probe, build_decoder_layer, model_preset
    from paper_2604_15379_b200.analytics import decode_step_bytes
    mach = b200_from_probe([74, 74])
    model = model_preset("qwen3-8b")
    g = build_decoder_layer(model, mach, "chiplet", 4, layers=36)
    m = report.metrics_algorithmic(g, ctx=1024, vocab=151936)
    want = decode_step_bytes(model, 4, 1024, 151936)
    assert m.hbm_read_bytes == want["total"]
    assert m.hbm_read_bytes_for(1) == want["kv"]
    assert math.isnan(m.l2_hit_rate)
    sc = report.stage_costs(g, 1024)
    assert len(sc) == len(g.stages) and all(s.flops == r.flops for s, r in zip(sc, g.stages))
