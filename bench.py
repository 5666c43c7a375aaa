"""Qwen3-8B decode benchmark of the B200 hierarchical task megakernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B]
                    [--mode chiplet_m_tile|chiplet_m_split|chiplet_n_major|standard]
                    [--impl ours|reference]

One step = one decode step of Qwen3-8B (36 layers + LM head + greedy argmax)
for ``batch`` sequences with a 1024-token KV context = one cooperative launch
of the persistent megakernel.  Weights are random-init bf16 (hash init, std
0.02), KV context synthetic bf16; weights (15.1 GB) exceed the 126 MB L2, so
no L2 flush is needed between steps.

Prints ONE JSON line (rank 0).  ``value`` = tokens/s with inputs resident in
HBM (device-timed with CUDA events over K back-to-back launches);
``e2e`` = the same metric through the public API with the step's token ids
copied host->device and the greedy ids device->host every step.
``--impl reference`` times the fp32 CPU oracle (oracle/qwen3_fp32.py, the
reference path restated; the reference package itself has no numerics) on a
bounded sample on the host cores.

Multi-GPU (torchrun): by default replicas -- every rank decodes its own
batch; value = all ranks' tokens / max-over-ranks time ("weak" scaling).
``--tp``: the ranks form one Megatron tensor-parallel group decoding ONE
batch (per-layer allreduces as device tasks over NVLink peer memory, CUDA
IPC bootstrap) -- "strong" scaling.  ``--tp-emulate N`` (1 GPU): N TP ranks
share the GPU on disjoint SM subsets (the device TP data path, measured).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
CTX = 1024
VOCAB = 151936


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out = self.proc.communicate(timeout=5)[0]
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for _, _, fl in rows for i, f in enumerate(fl)
                          if f.lower() == "active"})
        loaded = [r[0] for r in rows if r[0] > 0.5 * r[1]] or [r[0] for r in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def dist_setup(n_gpus):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    return rank, world, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def build(args, device):
    import torch
    from paper_2604_15379_b200 import MODES, b200_from_probe, build_decoder_layer, model_preset
    from paper_2604_15379_b200.analytics import device_tiles
    from paper_2604_15379_b200.runtime import Megakernel, halves_topology, probe, topology_summary
    from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights

    topo = probe(device)
    probe_ok = topo.num_dies == 2
    if not probe_ok:
        topo = halves_topology(topo.num_sms)
    graph_mode, trav, distn = MODES[args.mode]
    sched = "flat" if graph_mode == "standard" else "per_die"
    machine = b200_from_probe([topo.sms_per_die[i] for i in range(topo.num_dies)])
    model = model_preset("qwen3-8b")
    if args.layers != 36:
        from dataclasses import replace
        model = replace(model, num_layers=args.layers)
    g = build_decoder_layer(model, machine, graph_mode, args.batch,
                            tile_overrides=device_tiles(model, machine, graph_mode, args.batch,
                                                        t_m=args.t_m),
                            layers=model.num_layers)
    spec = Qwen3Spec.qwen3_8b(layers=model.num_layers)
    w = Qwen3Weights.random(spec, seed=0, device=f"cuda:{device}")
    t_max = CTX + 2 * (args.warmup + args.steps) + 64
    lm_tile = None
    if args.t_m is not None:
        from paper_2604_15379_b200.runtime import _default_lm_tile
        lm_tile = _default_lm_tile(spec, args.batch, args.t_m)
    mk = Megakernel(g, w, t_max=t_max, traversal=trav, distribution=distn, sched=sched,
                    topo=topo, keep_logits=False, device=device, lm_tile=lm_tile,
                    ksplit=not args.no_ksplit,
                    fuse_attn_reduce=os.environ.get("MK_FUSE_ATTN_REDUCE") == "1")
    del w
    torch.cuda.empty_cache()
    mk.fill_kv_random(CTX)
    if os.environ.get("MK_DEBUG"):
        mk.lib.mk_set_debug(mk.h, int(os.environ["MK_DEBUG"], 0))
    mk.set_tokens([(17 * i + 3) % VOCAB for i in range(args.batch)])
    info = {"topology": topology_summary(topo), "probe_ok": probe_ok, "graph_tasks": len(g.tasks),
            "units": len(mk.lowered.units)}
    return mk, model, spec, info


def run_ours(args):
    import torch
    from paper_2604_15379_b200.analytics import decode_step_bytes

    rank, world, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    mk, model, spec, info = build(args, local)
    B = args.batch
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        mk.launch()
    mk.sync()
    mk.reset_counters()
    barrier(world)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            mk.launch()
        ev1.record(stream)
        torch.cuda.synchronize()
    mk.sync()
    ms = ev0.elapsed_time(ev1)
    ctr = mk.counters()
    barrier(world)
    ms_max = max_over_ranks(ms, world)
    ms_step = ms_max / args.steps
    value = world * B * args.steps / (ms_max / 1e3)

    # e2e: public API, host tokens in / greedy tokens out every step
    h_tok = torch.tensor([(31 * i + 7) % VOCAB for i in range(B)], dtype=torch.int32).pin_memory()
    h_out = torch.empty(B, dtype=torch.int32).pin_memory()
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        # the C-ABI call with host buffers: H2D tokens, launch, D2H greedy ids
        mk.launch_host(h_tok, h_out, stream)
        e1.record(stream)
        e1.synchronize()
        h_tok.copy_(h_out)
    e2e_ms = e0.elapsed_time(e1)
    wall_ms = (time.perf_counter() - t0) * 1e3
    mk.sync()
    e2e_ms = max_over_ranks(max(e2e_ms, wall_ms), world)
    e2e_value = world * B * args.steps / (e2e_ms / 1e3)
    ok_tokens = bool(((h_out >= 0) & (h_out < VOCAB)).all())

    bytes_step = decode_step_bytes(model, B, CTX, VOCAB)
    peak, peak_kind = _peaks()
    achieved = bytes_step["total"] / (ms_step / 1e3) / 1e9
    traffic = _profiled_traffic(args)
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "tok/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (hash-init bf16 weights, synthetic 1024-token bf16 KV)",
        "config": {
            "workload": f"Qwen3-8B decode, batch {B}, ctx {CTX}, {args.mode} megakernel",
            "ksplit": not args.no_ksplit and args.mode != "standard",
            "t_m": next(t.tile_shape[0] for t in mk.graph.tasks if t.tile_shape),
            "batch_per_gpu": B, "ctx": CTX, "layers": model.num_layers, "mode": args.mode,
            "parallelism": "replicas" if world > 1 else "single",
            "l2": "no flush: 15.1 GB of weights per step >> 126 MB L2",
            "ms_per_token": round(ms_step, 4),
            **info,
        },
        "roofline": {
            "bound": "hbm",
            "achieved": round(achieved, 1),
            "peak": peak,
            "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "peak_kind": peak_kind,
            "frac_of_8TBs": round(achieved / 8000.0, 4),
            "algorithmic_bytes_per_step": bytes_step["total"],
            "traffic": traffic,
        },
        "e2e": {"value": round(e2e_value, 3), "unit": "tok/s",
                "h2d_bytes_per_step": 4 * B, "d2h_bytes_per_step": 4 * B,
                "ms_per_step": round(e2e_ms / args.steps, 4), "tokens_valid": ok_tokens},
        "gpu_launches": args.steps,
        "counters_per_step": {k: v // max(1, args.steps) for k, v in ctr.items() if k != "steps"},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    mk.close()


def build_tp(args, device, rank, world, emulate):
    """One Megakernel per TP rank: ``emulate`` = all ranks on this GPU (flat
    scheduler, #SMs / world CTAs each), else this process's rank on its own
    GPU (per-die scheduler) joined through CUDA IPC."""
    import torch
    from dataclasses import replace
    from paper_2604_15379_b200 import b200_from_probe, build_decoder_layer, model_preset
    from paper_2604_15379_b200 import dist as D
    from paper_2604_15379_b200.analytics import device_tiles
    from paper_2604_15379_b200.runtime import Megakernel, halves_topology, probe, topology_summary
    from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights
    topo = probe(device)
    if topo.num_dies != 2:
        topo = halves_topology(topo.num_sms)
    model = replace(model_preset("qwen3-8b"), num_layers=args.layers)
    spec = Qwen3Spec.qwen3_8b(layers=args.layers)
    w = Qwen3Weights.random(spec, seed=0, device=f"cuda:{device}")
    t_max = CTX + 2 * (args.warmup + args.steps) + 64
    if emulate:
        ctas = topo.num_sms // world
        mach = b200_from_probe([ctas])
        kw = dict(sched="flat", ctas=ctas, cooperative=False)
        ranks = range(world)
    else:
        mach = b200_from_probe([topo.sms_per_die[i] for i in range(topo.num_dies)])
        kw = dict(sched="per_die")
        ranks = [rank]
    g = build_decoder_layer(model, mach, "chiplet", args.batch,
                            tile_overrides=device_tiles(model, mach, "chiplet", args.batch,
                                                        tp=world), layers=args.layers)
    mks = [Megakernel(g, w, t_max=t_max, topo=topo, keep_logits=False, device=device,
                      tp=(r, world), **kw) for r in ranks]
    del w
    torch.cuda.empty_cache()
    if emulate:
        D.connect_local(mks)
    else:
        D.connect_dist(mks[0])
    for mk in mks:
        mk.fill_kv_random(CTX)
        mk.set_tokens([(17 * i + 3) % VOCAB for i in range(args.batch)])
    info = {"topology": topology_summary(topo), "graph_tasks": len(g.tasks),
            "units": len(mks[0].lowered.units), "tp": world,
            "tp_placement": f"{world} ranks on one GPU, {topo.num_sms // world} SMs each"
                            if emulate else "one rank per GPU (CUDA IPC peer regions)"}
    return mks, model, info


def run_tp(args):
    import torch
    from paper_2604_15379_b200.analytics import decode_step_bytes
    from paper_2604_15379_b200.dist import allreduce_bytes_per_step
    emulate = args.tp_emulate > 1
    rank, world, local = dist_setup(args.gpus) if not emulate else (0, 1, 0)
    tp = args.tp_emulate if emulate else world
    torch.cuda.set_device(local)
    mks, model, info = build_tp(args, local, rank, tp, emulate)
    streams = [torch.cuda.Stream() for _ in mks]
    main = torch.cuda.current_stream()

    def steps(n):
        ev = torch.cuda.Event()
        ev.record(main)
        for st in streams:
            st.wait_event(ev)
        for _ in range(n):
            for mk, st in zip(mks, streams):
                mk.launch(stream=st)
        for st in streams:
            e = torch.cuda.Event()
            e.record(st)
            main.wait_event(e)

    steps(args.warmup)
    for mk in mks:
        mk.sync()
    barrier(world)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(main)
        steps(args.steps)
        ev1.record(main)
        torch.cuda.synchronize()
    for mk in mks:
        mk.sync()
    ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    ms_step = ms / args.steps
    B = args.batch
    tokens = [mk.state.out_tokens.cpu() for mk in mks]
    same = all(torch.equal(t, tokens[0]) for t in tokens)
    bytes_step = decode_step_bytes(model, B, CTX, VOCAB)
    ar = allreduce_bytes_per_step(mks[0].spec, B, 4)
    line = {
        "metric": METRIC, "value": round(B / (ms_step / 1e3), 3), "unit": "tok/s",
        "n_gpus": 1 if emulate else world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (hash-init bf16 weights, synthetic 1024-token bf16 KV)",
        "config": {"workload": f"Qwen3-8B decode, batch {B}, ctx {CTX}, TP={tp} megakernel",
                   "parallelism": f"tp{tp}", "batch": B, "ctx": CTX, "layers": model.num_layers,
                   "ranks_agree_on_tokens": same,
                   "allreduce_fp32_bytes_per_step": ar["bytes_per_step"] * tp, **info},
        "roofline": {"bound": "hbm", "algorithmic_bytes_per_step": bytes_step["total"],
                     "achieved": round(bytes_step["total"] / (ms_step / 1e3) / 1e9, 1),
                     "unit": "GB/s (all ranks)"},
        "gpu_launches": args.steps * len(mks),
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    for mk in mks:
        mk.close()


def _profiled_traffic(args):
    """dram bytes per launch from a committed ncu --set full capture, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"{args.mode}_b{args.batch}")
    except Exception:
        return None


class CpuSample:
    """The fp32 CPU oracle (oracle/qwen3_fp32.py) on a bounded sample of the
    workload: ``sample_layers`` Qwen3-8B decoder layers at the same batch and
    1024-token context, plus the full-vocabulary LM-head GEMV.  A step is
    timed as  t(layers) * 36 / sample_layers + t(LM head)."""

    def __init__(self, batch: int, sample_layers: int = 2):
        import torch
        from oracle.qwen3_fp32 import Qwen3Fp32
        from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights
        self.threads = os.cpu_count() or 1
        torch.set_num_threads(self.threads)
        self.B, self.n = batch, sample_layers
        spec = Qwen3Spec.qwen3_8b(layers=sample_layers, vocab=1024)
        w = Qwen3Weights.random(spec, seed=0)
        self.o = Qwen3Fp32(w, t_max=CTX + 4, batch=batch)
        for li in range(sample_layers):
            self.o.k[li][:, :, :CTX].normal_()
            self.o.v[li][:, :, :CTX].normal_()
        self.head = torch.randn(VOCAB, spec.hidden)
        self.toks = torch.arange(batch) % 1024
        self.x = torch.randn(batch, spec.hidden)

    def step_seconds(self) -> float:
        self.o.pos[:] = CTX
        t0 = time.perf_counter()
        self.o.step(self.toks)
        t_layers = time.perf_counter() - t0
        t0 = time.perf_counter()
        (self.x @ self.head.T).argmax(-1)
        t_head = time.perf_counter() - t0
        return t_layers * (36 / self.n) + t_head

    def describe(self):
        return (f"fp32 torch oracle (oracle/qwen3_fp32.py): {self.n} of 36 Qwen3-8B layers at "
                f"batch {self.B}, ctx {CTX}, time x{36 // self.n} + timed 151936x4096 LM-head GEMV")


def cpu_baseline(args, sample_layers: int = 2):
    smp = CpuSample(args.batch, sample_layers)
    smp.step_seconds()                   # warm
    t = statistics.median(smp.step_seconds() for _ in range(3))
    return {"value": round(args.batch / t, 4), "unit": "tok/s", "cores": smp.threads,
            "kind": "port", "sample": smp.describe(), "ms_per_step": round(t * 1e3, 1)}


def run_reference(args):
    """The reference arm: the reference has no GPU path and no numerics
    (SURVEY.md section 0); its decode step restated as the fp32 CPU oracle,
    timed on the host cores on a bounded sample of the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t0 = time.perf_counter()
    smp = CpuSample(args.batch, sample_layers=1)
    for _ in range(args.warmup):
        smp.step_seconds()
    ts = [smp.step_seconds() for _ in range(args.steps)]
    t = statistics.median(ts)
    v = round(args.batch / t, 4)
    line = {
        "metric": METRIC, "value": v, "unit": "tok/s", "impl": "reference",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"Qwen3-8B decode, batch {args.batch}, ctx {CTX}, fp32 CPU oracle",
                   "batch_per_gpu": args.batch, "ctx": CTX},
        "cpu_baseline": {"value": v, "unit": "tok/s", "cores": smp.threads, "kind": "port",
                         "sample": smp.describe()},
        "e2e": {"value": v, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(time.perf_counter() - t0, 1),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layers", type=int, default=36)
    ap.add_argument("--mode", default="chiplet_m_tile",
                    choices=["chiplet_m_tile", "chiplet_m_split", "chiplet_n_major", "standard"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--t-m", type=int, default=None,
                    help="batch rows per m-tile (default: 16 for the GEMV body, "
                         "the whole batch up to 64 for tcgen05)")
    ap.add_argument("--tp", action="store_true",
                    help="torchrun ranks form one tensor-parallel group (default: replicas)")
    ap.add_argument("--tp-emulate", type=int, default=0,
                    help="N tensor-parallel ranks sharing this one GPU")
    ap.add_argument("--no-ksplit", action="store_true",
                    help="die tasks own whole tiles per schedule() (no K-split)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        if args.tp or args.tp_emulate > 1:
            run_tp(args)
        else:
            run_ours(args)


if __name__ == "__main__":
    main()
