"""chipletsim-compatible result records for device runs.

The reference turns one simulation into a ``SimTrace`` whose ``to_json()`` /
``csv_row()`` feed its CSV output and ``analytics.comparison_table``
(``/root/reference/pkg/src/chipletsim/runtime.py:59-71,92-171``,
``analytics.py:182-236``).  Here the same records are produced from a device
run:

* counters (fences, global / local atomics, polls, dispatches) come from the
  megakernel's own device counters (``mk_counters_get``);
* ``estimated_time_s`` is the *measured* device time per step (CUDA events);
* the memory metrics (L2 hit rate, HBM bytes) come from an ncu capture of the
  same launch when one is supplied (:func:`metrics_from_ncu`: the counters
  ``lts__t_sector_hit_rate.pct`` / ``lts__t_sectors_lookup_{hit,miss}.sum``,
  ``dram__bytes_{read,write}.sum``), else from the algorithmic bytes of the
  step (weights + KV, :func:`metrics_algorithmic`) with the L2 hit rate
  unknown (NaN) -- a device cannot read its L2 counters without a profiler;
* ``stages`` carry each stage's flops (the graph's ``StageRecord.flops``) and
  its algorithmic HBM bytes.

So ``comparison_table`` / ``comparison_json`` / ``compare`` accept device
traces exactly as they accept simulator traces.
"""

from __future__ import annotations

import csv
import io
import math
from dataclasses import dataclass, field

from .analytics import linear_gemm_dims
from .taskgraph import LINEAR_OPS, OpKind

SCHEMA_VERSION = 1

# ref runtime.py:59-71
CSV_COLUMNS = (
    "scenario_id",
    "mode",
    "batch",
    "l2_hit_rate",
    "hbm_read_bytes",
    "hbm_write_bytes",
    "fences",
    "global_atomics",
    "local_atomics",
    "dispatches",
    "est_time_s",
)

# ref memsim.py:50-56 (AccessRole order)
ROLES = ("weight", "activation", "output", "sync")


class CompareError(ValueError):
    """Traces are not comparable (ref runtime.py:80-81)."""


@dataclass(frozen=True)
class DeviceMetrics:
    """The ``Metrics`` fields the reference's reports read (memsim.py:150-200),
    from a measured capture or from algorithmic bytes.  ``source`` says which:
    "ncu" (measured), or "algorithmic" (L2 hit rate unknown = NaN)."""

    l2_hits: tuple = (0,)
    l2_misses: tuple = (0,)
    hbm_read_bytes_by_role: tuple = (0, 0, 0, 0)
    hbm_write_bytes_by_role: tuple = (0, 0, 0, 0)
    l2_hit_rate_measured: float | None = None
    source: str = "algorithmic"
    llc_hits: tuple = (0,)
    llc_misses: tuple = (0,)
    weight_rate: float | None = None    # role-attributed weight hit rate, when known

    @property
    def total_l2_hits(self) -> int:
        return sum(self.l2_hits)

    @property
    def total_l2_misses(self) -> int:
        return sum(self.l2_misses)

    @property
    def hbm_read_bytes(self) -> int:
        return sum(self.hbm_read_bytes_by_role)

    @property
    def hbm_write_bytes(self) -> int:
        return sum(self.hbm_write_bytes_by_role)

    def hbm_read_bytes_for(self, role) -> int:
        return self.hbm_read_bytes_by_role[int(role)]

    @property
    def l2_hit_rate(self) -> float:
        if self.l2_hit_rate_measured is not None:
            return self.l2_hit_rate_measured
        total = self.total_l2_hits + self.total_l2_misses
        return self.total_l2_hits / total if total else math.nan

    @property
    def weight_l2_hit_rate(self) -> float:
        if self.weight_rate is not None:
            return self.weight_rate
        # ncu does not attribute L2 lookups to roles; weights are >99% of the
        # sectors a decode step reads, so the overall rate stands in for it
        return self.l2_hit_rate


def _num(v: str) -> float:
    return float(v.replace(",", ""))


def metrics_from_ncu(text: str, kernel: str = "megakernel", launch: int = -1) -> DeviceMetrics:
    """Parse ``ncu --csv --metrics ...`` output (the "Metric Name" / "Metric
    Value" rows of one launch of ``kernel``; ``launch`` indexes the matching
    launches, default the last)."""
    rows = [r for r in csv.reader(io.StringIO(
        "\n".join(ln for ln in text.splitlines() if ln.startswith('"'))))]
    if not rows:
        raise ValueError("no ncu CSV rows")
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    need = ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")
    if any(k not in ix for k in need):
        raise ValueError(f"not an ncu --csv metrics table (header {hdr})")
    launches: dict = {}
    for r in rows[1:]:
        if len(r) < len(hdr) or kernel not in r[ix["Kernel Name"]]:
            continue
        launches.setdefault(r[ix["ID"]], {})[r[ix["Metric Name"]]] = (
            r[ix["Metric Unit"]], r[ix["Metric Value"]])
    if not launches:
        raise ValueError(f"no launch of {kernel!r} in the capture")
    m = launches[sorted(launches, key=int)[launch]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def bytes_of(name):
        if name not in m:
            return 0
        unit, val = m[name]
        return int(round(_num(val) * scale.get(unit, 1)))

    hits = int(_num(m["lts__t_sectors_lookup_hit.sum"][1])) \
        if "lts__t_sectors_lookup_hit.sum" in m else 0
    miss = int(_num(m["lts__t_sectors_lookup_miss.sum"][1])) \
        if "lts__t_sectors_lookup_miss.sum" in m else 0
    rate = None
    if "lts__t_sector_hit_rate.pct" in m:
        rate = _num(m["lts__t_sector_hit_rate.pct"][1]) / 100.0
    rd = bytes_of("dram__bytes_read.sum")
    wr = bytes_of("dram__bytes_write.sum")
    # ncu has no per-role split: reads are weights + KV (the step's streamed
    # operands), writes are outputs (activations, the appended KV rows)
    return DeviceMetrics(l2_hits=(hits,), l2_misses=(miss,),
                         hbm_read_bytes_by_role=(rd, 0, 0, 0),
                         hbm_write_bytes_by_role=(0, 0, wr, 0),
                         l2_hit_rate_measured=rate, source="ncu")


def kv_read_bytes(model, batch: int, ctx: int, layers: int | None = None) -> int:
    L = model.num_layers if layers is None else layers
    return batch * ctx * L * 2 * model.kv_heads * model.head_dim * model.dtype_bytes


def stage_bytes(g, ctx: int) -> list:
    """Algorithmic HBM bytes of every stage of ``g`` (weights streamed by its
    linear op, the KV cache its attention reads, the gammas of a norm)."""
    m = g.model
    dt = m.dtype_bytes
    out = []
    for s in g.stages:
        if s.op_kind in LINEAR_OPS:
            k, n = linear_gemm_dims(s.op_kind, m)
            b = k * n * dt
        elif s.op_kind == OpKind.ATTN_PARTIAL:   # KV + the q_norm / k_norm gammas
            b = kv_read_bytes(m, g.batch, ctx, layers=1) + 2 * m.head_dim * dt
        elif s.op_kind == OpKind.RMS_NORM:
            b = m.hidden_dim * dt
        else:
            b = 0
        out.append(b)
    return out


def metrics_algorithmic(g, ctx: int, vocab: int) -> DeviceMetrics:
    """Weights (every stage + final norm + LM head) as WEIGHT reads, the KV
    cache as ACTIVATION reads, the appended KV rows as OUTPUT writes."""
    m = g.model
    dt = m.dtype_bytes
    sb = stage_bytes(g, ctx)
    kv = sum(kv_read_bytes(m, g.batch, ctx, layers=1)
             for s in g.stages if s.op_kind == OpKind.ATTN_PARTIAL)
    w = sum(sb) - kv + m.hidden_dim * dt + vocab * m.hidden_dim * dt
    layers = len({s.layer for s in g.stages})
    kv_w = g.batch * layers * 2 * m.kv_heads * m.head_dim * dt
    return DeviceMetrics(hbm_read_bytes_by_role=(w, kv, 0, 0),
                         hbm_write_bytes_by_role=(0, 0, kv_w, 0))


@dataclass(frozen=True)
class StageCost:
    """ref runtime.py:84-89; ``hbm_bytes`` algorithmic."""
    name: str
    layer: int
    flops: int
    hbm_bytes: int


def stage_costs(g, ctx: int) -> tuple:
    return tuple(StageCost(s.name, s.layer, s.flops, b)
                 for s, b in zip(g.stages, stage_bytes(g, ctx)))


def trace_to_json(tr) -> dict:
    """Same keys as ``SimTrace.to_json`` (ref runtime.py:115-153)."""
    m = tr.metrics
    return {
        "schema_version": SCHEMA_VERSION,
        "mode": tr.mode,
        "batch": tr.batch,
        "traversal": tr.traversal,
        "distribution": tr.distribution,
        "steps": tr.steps,
        "l2_hit_rate": m.l2_hit_rate,
        "weight_l2_hit_rate": m.weight_l2_hit_rate,
        "l2_hits": list(m.l2_hits),
        "l2_misses": list(m.l2_misses),
        "llc_hits": list(m.llc_hits),
        "llc_misses": list(m.llc_misses),
        "hbm_read_bytes": m.hbm_read_bytes,
        "hbm_write_bytes": m.hbm_write_bytes,
        "hbm_read_bytes_by_role": dict(zip(ROLES, m.hbm_read_bytes_by_role)),
        "hbm_write_bytes_by_role": dict(zip(ROLES, m.hbm_write_bytes_by_role)),
        "fences": tr.fences_issued,
        "fence_flush_lines": getattr(tr, "fence_flush_lines", 0),
        "global_atomics": tr.global_atomics,
        "local_atomics": tr.local_atomics,
        "polls": tr.poll_count,
        "dispatches": tr.dispatches,
        "stages": [{"name": s.name, "layer": s.layer, "flops": s.flops,
                    "hbm_bytes": s.hbm_bytes} for s in tr.stage_costs],
        "estimated_time_s": tr.estimated_time_s,
        "policy": list(tr.policy_notes),
    }


def trace_csv_row(tr, scenario_id: str) -> str:
    """ref runtime.py:155-171 (CSV_COLUMNS order)."""
    m = tr.metrics
    return ",".join((
        scenario_id, tr.mode, str(tr.batch), f"{m.l2_hit_rate:.6f}",
        str(m.hbm_read_bytes), str(m.hbm_write_bytes), str(tr.fences_issued),
        str(tr.global_atomics), str(tr.local_atomics), str(tr.dispatches),
        f"{tr.estimated_time_s:.9e}"))


def csv_text(rows) -> str:
    """Header + one row per ``(scenario_id, trace)``."""
    return "\n".join([",".join(CSV_COLUMNS)] +
                     [trace_csv_row(t, sid) for sid, t in rows]) + "\n"


def _ratio(b, a):
    if a == 0:
        return 1.0 if b == 0 else float("inf")
    return b / a


@dataclass(frozen=True)
class ComparisonReport:
    """ref runtime.py:551-570."""
    baseline: object
    candidate: object
    ratios: dict = field(default_factory=dict)

    def to_json(self) -> dict:
        return {"schema_version": SCHEMA_VERSION,
                "baseline_mode": self.baseline.mode,
                "candidate_mode": self.candidate.mode,
                "batch": self.baseline.batch,
                "ratios": dict(self.ratios),
                "baseline_weight_hit_rate": self.baseline.metrics.weight_l2_hit_rate,
                "candidate_weight_hit_rate": self.candidate.metrics.weight_l2_hit_rate}


def compare(a, b) -> ComparisonReport:
    """ref runtime.py:579-602 for device traces (same workload, two policies)."""
    if a.batch != b.batch or a.model_fingerprint != b.model_fingerprint:
        raise CompareError("traces come from different model/batch configs")
    ma, mb = a.metrics, b.metrics
    ratios = {
        "l2_hit_rate": _ratio(mb.l2_hit_rate, ma.l2_hit_rate),
        "weight_l2_hit_rate": _ratio(mb.weight_l2_hit_rate, ma.weight_l2_hit_rate),
        "hbm_read_bytes": _ratio(mb.hbm_read_bytes, ma.hbm_read_bytes),
        "hbm_write_bytes": _ratio(mb.hbm_write_bytes, ma.hbm_write_bytes),
        "hbm_weight_read_bytes": _ratio(mb.hbm_read_bytes_for(0), ma.hbm_read_bytes_for(0)),
        "fences": _ratio(b.fences_issued, a.fences_issued),
        "global_atomics": _ratio(b.global_atomics, a.global_atomics),
        "local_atomics": _ratio(b.local_atomics, a.local_atomics),
        "dispatches": _ratio(b.dispatches, a.dispatches),
        "est_time_s": _ratio(b.estimated_time_s, a.estimated_time_s),
    }
    return ComparisonReport(a, b, ratios)


def comparison_table(rows, baseline_mode: str = "standard") -> str:
    """Per-mode L2 hit rate and HBM traffic normalised to ``baseline_mode``
    (ref analytics.py:182-213); ``rows`` = ``[(batch, {mode: trace})]`` of
    device or simulator traces."""
    rows = list(rows)
    if not rows:
        return "(no results)\n"
    modes = list(rows[0][1])
    others = [m for m in modes if m != baseline_mode]
    header = (["BS"] + [f"L2Hit% {m}" for m in modes]
              + [f"HBMRd x{baseline_mode} {m}" for m in others]
              + [f"HBMWr x{baseline_mode} {m}" for m in others])
    lines = ["  ".join(f"{h:>22}" for h in header)]
    for batch, by_mode in rows:
        base = by_mode.get(baseline_mode)
        cells = [f"{batch:>22}"]
        cells += [f"{by_mode[m].metrics.l2_hit_rate * 100:>21.1f}%" for m in modes]
        for kind in ("hbm_read_bytes", "hbm_write_bytes"):
            for m in others:
                val = getattr(by_mode[m].metrics, kind)
                ref = getattr(base.metrics, kind) if base else 0
                cells.append(f"{(val / ref if ref else float('nan')):>22.2f}")
        lines.append("  ".join(cells))
    return "\n".join(lines) + "\n"


def comparison_json(rows, baseline_mode: str = "standard") -> dict:
    """JSON form of :func:`comparison_table` (ref analytics.py:216-236)."""
    out = {"schema_version": 1, "baseline_mode": baseline_mode, "rows": []}
    for batch, by_mode in rows:
        base = by_mode.get(baseline_mode)
        entry = {"batch": batch, "modes": {}}
        for m, trace in by_mode.items():
            met = trace.metrics
            rec = {"l2_hit_rate": met.l2_hit_rate,
                   "weight_l2_hit_rate": met.weight_l2_hit_rate,
                   "hbm_read_bytes": met.hbm_read_bytes,
                   "hbm_write_bytes": met.hbm_write_bytes,
                   "est_time_s": trace.estimated_time_s}
            if base is not None and m != baseline_mode:
                bm = base.metrics
                rec["hbm_read_vs_baseline"] = (met.hbm_read_bytes / bm.hbm_read_bytes
                                               if bm.hbm_read_bytes else None)
                rec["hbm_write_vs_baseline"] = (met.hbm_write_bytes / bm.hbm_write_bytes
                                                if bm.hbm_write_bytes else None)
            entry["modes"][m] = rec
        out["rows"].append(entry)
    return out
