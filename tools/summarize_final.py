"""Summarise a tools/final_measure.sh pass into profiles/<round>/.

    python tools/summarize_final.py gpurun_out/final profiles/r01b

Copies the bench JSON lines, writes a markdown table of the sweep (die-aware
vs flat, ablations), the ncu full-set summaries of the B=1 / B=64 megakernel
launch, the L2-hit / DRAM-byte comparison and the launch list, and updates
profiles/ncu_traffic.json (the `roofline.traffic` source of bench.py).
"""
import csv
import glob
import io
import json
import os
import shutil
import sys

SRC, DST = sys.argv[1], sys.argv[2]
os.makedirs(DST, exist_ok=True)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(tag):
    try:
        with open(os.path.join(SRC, f"{tag}.json")) as f:
            return json.loads(f.read().strip().splitlines()[-1])
    except Exception:
        return None


# ---- bench lines -----------------------------------------------------------
for path in glob.glob(os.path.join(SRC, "*.json")):
    shutil.copy(path, DST)
rows = []
tags = sorted({os.path.basename(p)[:-5] for p in glob.glob(os.path.join(SRC, "b[0-9]*.json"))},
              key=lambda t: (int(t.split("_")[0][1:]), t))
for t in tags:
    d = load(t)
    if not d:
        continue
    rows.append((t, d["config"]["batch_per_gpu"], d["config"]["mode"], d["config"].get("t_m"),
                 d["config"].get("ksplit"), d["ms_per_step"], d["value"], d["roofline"]["frac"],
                 d["roofline"]["frac_of_8TBs"], d["e2e"]["value"]))
with open(os.path.join(DST, "sweep.md"), "w") as f:
    f.write("# Bench sweep (1x B200, Qwen3-8B decode, ctx 1024, bf16, synthetic weights)\n\n")
    f.write("`python bench.py --batch B [--mode M] [--t-m T] [--no-ksplit] --steps 10 --warmup 3`; "
            "device time over 10 launches (CUDA events), 36 layers + LM head + argmax per step.\n\n")
    f.write("| tag | batch | mode | T_M | K-split | ms/step | tok/s | HBM frac (measured peak) | frac of 8 TB/s | e2e tok/s |\n")
    f.write("|---|---|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        f.write("| " + " | ".join(str(x) for x in r) + " |\n")
    # die-aware vs flat
    f.write("\n## Die-aware (chiplet_m_tile) vs die-unaware flat megakernel (standard)\n\n")
    f.write("| batch | die-aware ms | flat ms | speed-up |\n|---|---|---|---|\n")
    for b in (1, 8, 32, 64):
        a, s = load(f"b{b}_m_tile"), load(f"b{b}_standard")
        if a and s:
            f.write(f"| {b} | {a['ms_per_step']} | {s['ms_per_step']} | "
                    f"{s['ms_per_step'] / a['ms_per_step']:.2f}x |\n")
    f.write("\n## Paper ablation at the paper's tiles (T_M = 16: cooperative m-tiles)\n\n")
    f.write("| batch | M-tile ms | M-split ms | flat ms | M-tile vs M-split | M-tile vs flat |\n|---|---|---|---|---|---|\n")
    for b in (32, 64):
        a, m, s = load(f"b{b}_m_tile_tm16"), load(f"b{b}_m_split_tm16"), load(f"b{b}_standard_tm16")
        if a and m and s:
            f.write(f"| {b} | {a['ms_per_step']} | {m['ms_per_step']} | {s['ms_per_step']} | "
                    f"{m['ms_per_step'] / a['ms_per_step']:.2f}x | {s['ms_per_step'] / a['ms_per_step']:.2f}x |\n")

# ---- ncu full-set summaries -------------------------------------------------
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
traffic = {}
for tag in ("b1", "b8", "b16", "b64"):
    path = os.path.join(SRC, f"ncu_{tag}_raw.csv")
    if not os.path.exists(path):
        continue
    rows = list(csv.reader(open(path)))
    h, units, v = rows[0], rows[1], rows[2]
    got = {n: (units[i], v[i]) for i, n in enumerate(h)}
    stalls = sorted(((n, float(v[i])) for i, n in enumerate(h)
                     if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")
                     and v[i] not in ("", "n/a")), key=lambda x: -x[1])
    tot = sum(x for _, x in stalls) or 1.0
    with open(os.path.join(DST, f"ncu_{tag}_summary.md"), "w") as f:
        f.write(f"# ncu --set full: one megakernel launch, Qwen3-8B decode {tag.upper()}, chiplet_m_tile\n\n")
        f.write(f"`ncu --set full --import-source on --clock-control none -k regex:megakernel -s 4 -c 1 "
                f"python bench.py --batch {tag[1:]} --steps 2 --warmup 3 --no-cpu-baseline`\n\n")
        f.write("| metric | unit | value |\n|---|---|---|\n")
        for n in WANT:
            if n in got:
                f.write(f"| {n} | {got[n][0]} | {got[n][1]} |\n")
        f.write("\n| stall reason (all warps incl. spinning roles) | share |\n|---|---|\n")
        for n, x in stalls[:10]:
            f.write(f"| {n.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {100 * x / tot:.1f}% |\n")
    try:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(got["dram__bytes_read.sum"][1]) * scale[got["dram__bytes_read.sum"][0]]
        wr = float(got["dram__bytes_write.sum"][1]) * scale[got["dram__bytes_write.sum"][0]]
        traffic[f"chiplet_m_tile_{tag}"] = int(rd + wr)
    except Exception:
        pass

# ---- L2 / DRAM comparison ----------------------------------------------------
def metrics(tag):
    path = os.path.join(SRC, f"l2_{tag}.csv")
    if not os.path.exists(path):
        return None
    text = open(path).read()
    start = text.find('"ID"')
    if start < 0:
        return None
    out = {}
    for r in csv.DictReader(io.StringIO(text[start:])):
        out[r["Metric Name"]] = (r["Metric Unit"], r["Metric Value"])
    return out


with open(os.path.join(DST, "l2_dram.md"), "w") as f:
    f.write("# L2 hit rate and DRAM bytes per step: die-aware vs flat (ncu, one launch after warm-up)\n\n")
    f.write("| config | time | DRAM read | DRAM write | HBM B/token | L2 hit % | DRAM throughput % |\n|---|---|---|---|---|---|---|\n")
    for tag in ("b1_m_tile", "b1_standard", "b32_m_tile", "b32_standard", "b64_m_tile", "b64_standard",
                "b64_m_tile_tm16", "b64_standard_tm16"):
        m = metrics(tag)
        if not m:
            continue
        b = int(tag.split("_")[0][1:])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        try:
            rd = float(m["dram__bytes_read.sum"][1].replace(",", "")) * scale[m["dram__bytes_read.sum"][0]]
            wr = float(m["dram__bytes_write.sum"][1].replace(",", "")) * scale[m["dram__bytes_write.sum"][0]]
            per_tok = f"{(rd + wr) / b / 1e9:.3f} GB"
        except Exception:
            per_tok = "?"
        g = lambda k: " ".join(m.get(k, ("", "?"))[::-1])
        f.write(f"| {tag} | {g('gpu__time_duration.sum')} | {g('dram__bytes_read.sum')} | "
                f"{g('dram__bytes_write.sum')} | {per_tok} | {g('lts__t_sector_hit_rate.pct')} | "
                f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} |\n")

# ---- launch list -------------------------------------------------------------
path = os.path.join(SRC, "launches_b1.csv")
if os.path.exists(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:]))) if start >= 0 else []
    mk = [float(r["Metric Value"].replace(",", "")) for r in rows
          if "megakernel" in r["Kernel Name"] and r["Metric Name"] == "gpu__time_duration.sum"]
    allk = [float(r["Metric Value"].replace(",", "")) for r in rows if r["Metric Name"] == "gpu__time_duration.sum"]
    unit = rows[0]["Metric Unit"] if rows else ""
    with open(os.path.join(DST, "launches_b1.md"), "w") as f:
        f.write("# Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none "
                "python bench.py --steps 3 --warmup 3 --no-cpu-baseline` (B=1)\n\n")
        f.write(f"Whole process: {len(allk)} kernel launches (weight init / packing run once at start-up); "
                f"megakernel launches: {len(mk)} (one per decode step, incl. warm-up and the e2e pass).\n\n")
        f.write(f"megakernel per launch ({unit}, cold-cache and serialised under ncu): "
                + ", ".join(f"{x:.0f}" for x in mk) + "\n\n")
        f.write("Inside the timed region of bench.py only the megakernel runs (`gpu_launches` = steps).\n")

if traffic:
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        cur = json.load(open(tp))
    except Exception:
        cur = {}
    cur.update(traffic)
    cur["_source"] = f"{DST}/ncu_*_summary.md: dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full)"
    json.dump(cur, open(tp, "w"), indent=1)
print("wrote", DST)
