"""Reference-simulator sync counters over a sweep of workers-per-die W
(test infrastructure; run in the build container, where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python oracle/gen_sim_w.py

The device probe splits a B200 into dies of 68/80 .. 74/74 SMs depending on
the part, so the uniform W the reference needs (ref machine.py:119-128) is
the smaller die minus its scheduler SM.  For every W in 64..77 this runs the
reference's own ``simulate`` (ref runtime.py:253-548) on

* the toy 2-layer chiplet graph at B=2 (the device test's graph), and
* one Qwen3-8B chiplet decoder layer at B=1 with the device GEMV tiles,

and records dispatches / fences / global and local atomics in
``tests/golden/sim_counters_w.json``.  ``oracle/sched_accounting.py`` is
pinned to these numbers (tests/test_oracle_sched.py), and the device
counters are checked against the restatement at the probed W, 36 layers
(tests/test_gpu_megakernel.py).
"""

from __future__ import annotations

import dataclasses
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


def main():
    base = ref_machine.load_machine(OUT / "b200_machine.json")
    from paper_2604_15379_b200 import analytics as ours
    from paper_2604_15379_b200 import machine as ours_m
    recs = []
    for W in range(64, 78):
        mach = dataclasses.replace(base, cus_per_xcd=W + 1, workers_per_xcd=W)
        for model_name, batch, layers in (("toy", 2, 2), ("qwen3-8b", 1, 1)):
            model = ref_machine.model_preset(model_name)
            if model_name == "toy":
                tiles = ref_scenario.fit_tiles(model, mach, "chiplet")
            else:
                om = ours_m.model_preset(model_name)
                omach = ours_m.b200_from_probe([W + 1, W + 1])
                raw = ours.device_tiles(om, omach, "chiplet", batch)
                tiles = {(k if k == "silu_chunk" else ref_tg.OpKind(k.value)): v
                         for k, v in raw.items()}
            g = ref_tg.build_decoder_layer(model, mach, "chiplet", batch,
                                           tile_overrides=tiles, layers=layers)
            tr = ref.simulate(g, mach, traversal=ref_tr.Traversal.M_MAJOR_WINDOWED,
                              distribution=ref_tr.Distribution.M_TILE)
            rec = dict(workers=W, model=model_name, mode="chiplet", batch=batch,
                       layers=layers, tiles="fit" if model_name == "toy" else "device",
                       dispatches=tr.dispatches, fences=tr.fences_issued,
                       global_atomics=tr.global_atomics,
                       local_atomics=tr.local_atomics)
            recs.append(rec)
            print(rec, flush=True)
    (OUT / "sim_counters_w.json").write_text(json.dumps(recs, indent=0) + "\n")


if __name__ == "__main__":
    main()
