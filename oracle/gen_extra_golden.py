"""Golden payload / flops digests and GraphError messages from the REFERENCE
(test infrastructure; build container only).

* ``payloads.json``: per graph case, the sha256 of every task's (id, payload
  class, payload fields, flops, stage) and every stage's flops -- the part of
  a TaskGraph that graph_to_json leaves out (ref taskgraph.py:73-112, 647-682);
* ``graph_errors.json``: the reference's GraphError message for each
  malformed graph of oracle/graph_mutations.py and each bad builder call.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python oracle/gen_extra_golden.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

from chipletsim import machine as rm  # noqa: E402  (reference, via PYTHONPATH)
from chipletsim import taskgraph as rt

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
from oracle.gen_extra_golden_doc import digest, payload_doc  # noqa: E402
from oracle.graph_mutations import BUILD_ERRORS, MUTATIONS  # noqa: E402

CASES = [dict(machine=m, model=mo, mode=md, batch=b, layers=ly)
         for m, mo, ly in (("b200", "toy", 2), ("b200", "qwen3-8b", 1), ("mi350", "qwen3-8b", 1))
         for md in ("standard", "chiplet") for b in (1, 8, 33)]


def machine_of(name, mod):
    return mod.load_machine(GOLD / "b200_machine.json") if name == "b200" else mod.preset(name)


def main():
    pays = []
    for c in CASES:
        g = rt.build_decoder_layer(rm.model_preset(c["model"]), machine_of(c["machine"], rm),
                                   c["mode"], c["batch"], layers=c["layers"])
        pays.append(dict(c, n_tasks=len(g.tasks), sha256=digest(payload_doc(g))))
    (GOLD / "payloads.json").write_text(json.dumps(pays, indent=0) + "\n")
    errs = {}
    mach = rm.preset("toy")
    base = rt.build_decoder_layer(rm.model_preset("toy"), mach, "chiplet", 2, layers=2)
    for name, fn in MUTATIONS.items():
        try:
            rt.validate_graph(fn(base))
            errs[name] = None
        except rt.GraphError as e:
            errs[name] = str(e)
    for name, kw in BUILD_ERRORS.items():
        try:
            rt.build_decoder_layer(rm.model_preset("toy"), mach, kw["mode"], kw["batch"],
                                   layers=kw["layers"])
            errs[name] = None
        except rt.GraphError as e:
            errs[name] = str(e)
    (GOLD / "graph_errors.json").write_text(json.dumps(errs, indent=1) + "\n")
    print(json.dumps(errs, indent=1))


if __name__ == "__main__":
    main()
