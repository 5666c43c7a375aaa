"""Golden reference reports (test infrastructure): the REFERENCE's own
``SimTrace.to_json()``, ``csv_row()``, ``compare().to_json()`` and
``analytics.comparison_table`` / ``comparison_json`` for toy-layer
simulations, with the metric numbers they were computed from.
``tests/test_report.py`` feeds the same numbers through
``paper_2604_15379_b200.report`` and requires identical records / text.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python oracle/gen_report_golden.py
"""

from __future__ import annotations

import json
from pathlib import Path

import chipletsim as ref  # noqa: E402  (reference, via PYTHONPATH)
from chipletsim import analytics as ref_an
from chipletsim import machine as ref_machine
from chipletsim import runtime as ref_rt
from chipletsim import taskgraph as ref_tg

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden" / "reports.json"


def main():
    mach = ref_machine.preset("toy")
    model = ref_machine.model_preset("toy")
    traces = {}
    rows = []
    for batch in (1, 8):
        by_mode = {}
        for mode in ("standard", "chiplet"):
            g = ref_tg.build_decoder_layer(model, mach, mode, batch)
            tr = ref.simulate(g, mach)
            by_mode[mode] = tr
            m = tr.metrics
            traces[f"{mode}_b{batch}"] = dict(
                to_json=tr.to_json(), csv_row=tr.csv_row(f"{mode}_b{batch}"),
                numbers=dict(l2_hits=list(m.l2_hits), l2_misses=list(m.l2_misses),
                             hbm_read_bytes_by_role=list(m.hbm_read_bytes_by_role),
                             hbm_write_bytes_by_role=list(m.hbm_write_bytes_by_role),
                             weight_l2_hit_rate=m.weight_l2_hit_rate))
        rows.append((batch, by_mode))
    doc = dict(csv_columns=list(ref_rt.CSV_COLUMNS), traces=traces,
               comparison_table=ref_an.comparison_table(rows),
               comparison_json=ref_an.comparison_json(rows),
               compare=ref_rt.compare(rows[1][1]["standard"], rows[1][1]["chiplet"]).to_json())
    OUT.write_text(json.dumps(doc, indent=0) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
