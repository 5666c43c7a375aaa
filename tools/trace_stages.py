"""Per-stage phase breakdown of one decode step from the per-unit trace
(mk_trace_enable): for every stage, over the units of one representative
layer range, the distribution of
  wait   = dependency acquired - poll start (idle on the input event)
  stage  = body start - acquired          (operand staging: x / norm)
  body   = consumer-0 done - body start   (streaming + math)
  skew   = all consumers done - consumer-0 done
  signal = signalled - all consumers done
and the stage span (first acquire -> last signal).

    python tools/trace_stages.py --batch 1 [--mode chiplet_m_tile] [--layers 36]
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layers", type=int, default=36)
    ap.add_argument("--mode", default="chiplet_m_tile")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--t-m", type=int, default=None)
    ap.add_argument("--no-ksplit", action="store_true")
    ap.add_argument("--out", default="gpurun_out/trace.json")
    ap.add_argument("--detail", action="append", default=[],
                    help="stage key (e.g. L17.qkv): per-worker rows of that stage")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    mk, model, spec, info = bench.build(args, 0)
    for _ in range(3):
        mk.launch()
    mk.sync()
    cap = 4096
    mk.enable_trace(cap)
    mk.launch()
    mk.sync()
    tr = mk.read_trace()
    names = mk.lowered.task_names
    gw_of = np.repeat(np.arange(tr.shape[0]), tr.shape[1])
    recs = tr.reshape(-1, 8)
    keep = recs[:, 7] > 0
    recs, gw_of = recs[keep], gw_of[keep]
    t0 = int(recs[:, 2].min())
    by = collections.OrderedDict()
    order = []
    for r in recs[np.argsort(recs[:, 2], kind="stable")]:
        task = int(r[0] & 0xFFFFFFFF)
        nm = names[task]
        key = nm.rsplit(".", 1)[0] if nm.startswith("L") else nm.split(".")[0]
        if key not in by:
            order.append(key)
        by.setdefault(key, []).append(r.astype(np.int64))
    rows = []
    for key in order:
        rs = np.array(by[key])
        wait = (rs[:, 2] - rs[:, 1]) / 1e3
        body_start = np.where(rs[:, 3] > 0, rs[:, 3], rs[:, 2])
        stage = (body_start - rs[:, 2]) / 1e3
        body = (rs[:, 4] - body_start) / 1e3
        skew = (rs[:, 5] - rs[:, 4]) / 1e3
        sig = (rs[:, 6] - rs[:, 5]) / 1e3
        # sub-phases packed in word 7: consumers released / x rows loaded (ns after acquire)
        rel = ((rs[:, 7] >> 20) & 0x3FFFFF) / 1e3
        xld = ((rs[:, 7] >> 42) & 0x3FFFFF) / 1e3
        rows.append(dict(stage=key, units=len(rs),
                         start=(rs[:, 2].min() - t0) / 1e3, end=(rs[:, 6].max() - t0) / 1e3,
                         first_done=(rs[:, 6].min() - t0) / 1e3,
                         wait_med=float(np.median(wait)), stage_med=float(np.median(stage)),
                         body_med=float(np.median(body)), body_max=float(body.max()),
                         body_min=float(body.min()),
                         skew_med=float(np.median(skew)), sig_med=float(np.median(sig)),
                         sig_max=float(sig.max()),
                         rel_med=float(np.median(rel)),
                         xld_med=float(np.median(xld[xld > 0])) if (xld > 0).any() else 0.0))
    total = (recs[:, 6].max() - t0) / 1e3
    print(f"total {total:.1f} us")
    hdr = ("stage", "units", "start", "end", "1st_done", "stage_med", "body_min", "body_med",
           "body_max", "skew_med", "sig_med", "sig_max", "rel_med", "xld_med")
    print(" ".join(f"{h:>10}" for h in hdr))
    for r in rows:
        if r["stage"].startswith(("L0.", "L1.", "L17.", "L35.")) or not r["stage"].startswith("L"):
            print(f"{r['stage']:>10} {r['units']:>10} " + " ".join(
                f"{r[k]:>10.2f}" for k in ("start", "end", "first_done", "stage_med", "body_min",
                                           "body_med", "body_max", "skew_med", "sig_med",
                                           "sig_max", "rel_med", "xld_med")))
    W = mk.lowered.workers
    for key in args.detail:
        sel = [i for i in range(len(recs))
               if names[int(recs[i, 0] & 0xFFFFFFFF)].startswith(key + ".")]
        if not sel:
            continue
        t_first = min(int(recs[i, 2]) for i in sel)
        rows_d = []
        for i in sel:
            r = recs[i].astype(np.int64)
            bs = r[3] if r[3] > 0 else r[2]
            rows_d.append((gw_of[i] // W, gw_of[i] % W, (r[2] - t_first) / 1e3, (bs - r[2]) / 1e3,
                           (r[4] - bs) / 1e3, (r[6] - t_first) / 1e3,
                           ((r[7] >> 20) & 0x3FFFFF) / 1e3, ((r[7] >> 42) & 0x3FFFFF) / 1e3,
                           names[int(r[0] & 0xFFFFFFFF)]))
        rows_d.sort(key=lambda x: -x[4])
        print(f"-- {key}: slowest bodies (die, worker, acquired, stage, body, signalled, "
              "stamp6, stamp7 [after acquire], task)")
        for d in rows_d[:12]:
            print("   die %d w %3d  acq %6.2f  stage %5.2f  body %6.2f  sig %6.2f  s6 %6.2f  s7 %6.2f  %s" % d)
        for die in sorted({d[0] for d in rows_d}):
            b = np.array([d[4] for d in rows_d if d[0] == die])
            print(f"   die {die}: n={len(b)} body med {np.median(b):.2f} max {b.max():.2f}")
        wb = sorted(rows_d, key=lambda x: (x[0], x[1]))
        print("   body by worker:", " ".join(f"{d[4]:.0f}" for d in wb))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(dict(batch=args.batch, mode=args.mode, total_us=total, stages=rows, **info),
              open(args.out, "w"), indent=1)
    mk.close()


if __name__ == "__main__":
    main()
