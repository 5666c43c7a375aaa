"""Payload digest helpers shared by oracle/gen_extra_golden.py (which runs
the reference) and tests/test_api_parity.py (which runs this package): test
infrastructure, no reference import."""

import dataclasses
import hashlib
import json


def _plain(v):
    if dataclasses.is_dataclass(v):
        return {f.name: _plain(getattr(v, f.name)) for f in dataclasses.fields(v)}
    if isinstance(v, (tuple, list)):
        return [_plain(x) for x in v]
    if hasattr(v, "value") and not isinstance(v, (int, float, str)):
        return v.value
    return v


def payload_doc(g):
    return {"tasks": [[t.id, type(t.work).__name__, _plain(t.work), t.flops, t.stage]
                      for t in g.tasks],
            "stages": [[s.name, s.layer, s.flops] for s in g.stages]}


def digest(doc):
    return hashlib.sha256(json.dumps(doc).encode()).hexdigest()
