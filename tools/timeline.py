"""Per-stage timeline of one Qwen3-8B decode step from the device event log.

    python tools/timeline.py --batch 1 --mode chiplet_m_tile [--layers 36]

Prints, per stage of one representative layer (and totals): first start,
last end, span, and the busy time distribution over workers, plus the gaps
between consecutive stages (dependency latency).
"""

import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layers", type=int, default=36)
    ap.add_argument("--mode", default="chiplet_m_tile")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    ap.add_argument("--t-m", type=int, default=None)
    ap.add_argument("--no-ksplit", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    mk, model, spec, info = bench.build(args, 0)
    for _ in range(3):
        mk.launch()
    mk.sync()
    cap = 1 << 21
    mk.enable_log(cap)
    mk.launch()
    mk.sync()
    recs, n = mk.read_log(cap)
    names = mk.lowered.task_names
    exe = [r for r in recs if r.kind == 1]
    phases = {}
    for r in recs:
        if r.kind in (2, 3, 4, 5):
            phases.setdefault(r.kind, []).append((r.t_end - r.t_start) / 1e3)
    for k, name in ((2, "attn prologue"), (3, "attn K/V slot wait"), (4, "attn token loop"),
                    (5, "attn merge")):
        v = phases.get(k, [])
        if v:
            v.sort()
            print(f"{name:>20}: n {len(v)} mean {sum(v)/len(v):.2f} us  p50 {v[len(v)//2]:.2f}  max {v[-1]:.2f}")
    disp = [r for r in recs if r.kind == 0]
    t0 = min(r.t_start for r in exe)
    stage = collections.OrderedDict()
    for r in exe:
        nm = names[r.task]
        key = nm.rsplit(".", 1)[0] if nm.startswith("L") else nm.split(".")[0]
        stage.setdefault(key, []).append(r)
    rows = []
    prev_end = None
    for key, rs in stage.items():
        s = min(r.t_start for r in rs) - t0
        e = max(r.t_end for r in rs) - t0
        busy = [r.t_end - r.t_start for r in rs]
        rows.append({"stage": key, "start_us": s / 1e3, "end_us": e / 1e3,
                     "span_us": (e - s) / 1e3,
                     "gap_us": None if prev_end is None else (s - prev_end) / 1e3,
                     "units": len(rs), "busy_max_us": max(busy) / 1e3,
                     "busy_mean_us": sum(busy) / len(busy) / 1e3})
        prev_end = e
    total = (max(r.t_end for r in exe) - t0) / 1e3
    sched_span = (max(r.t_end for r in disp) - min(r.t_start for r in disp)) / 1e3
    out = {"batch": args.batch, "mode": args.mode, "total_us": total,
           "sched_dispatch_span_us": sched_span, "stages": rows}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(f"total {total:.1f} us, scheduler dispatch span {sched_span:.1f} us")
    for r in rows[:20] + rows[-12:]:
        print(f"{r['stage']:>22} start {r['start_us']:9.1f} span {r['span_us']:8.1f} "
              f"gap {r['gap_us'] if r['gap_us'] is None else round(r['gap_us'],1)!s:>7} "
              f"units {r['units']:5d} busy max {r['busy_max_us']:7.1f} mean {r['busy_mean_us']:7.1f}")
    mk.close()


if __name__ == "__main__":
    main()
