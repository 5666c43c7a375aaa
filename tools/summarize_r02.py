"""Markdown summary of a round-2 measurement directory (tools/r02_final2.sh
output copied under profiles/r02/<dir>/).

    python tools/summarize_r02.py profiles/r02/final3 > profiles/r02/final3/README.md
"""
import csv
import glob
import io
import json
import os
import sys


def J(d, name):
    return json.loads(open(os.path.join(d, name)).read().strip().splitlines()[-1])


def main():
    d = sys.argv[1]
    top = J(d, "bench_default.json")["config"]["topology"]
    b = J(d, "bench_default.json")
    r = J(d, "bench_reference.json")
    print(f"# Round-2 measurement pass ({os.path.basename(d)}: one B200, {top['sms_per_die']} SMs per die, "
          f"W = {min(top['sms_per_die']) - 1} workers per die)\n")
    print(f"SM clock {b['clocks']['sm_mhz']} / {b['clocks']['sm_max_mhz']} MHz, throttle reasons {b['clocks']['reasons']}.\n")
    print("## Headline (`python bench.py`, B=1, ctx 1024, 36 layers + LM head + argmax)\n")
    print(f"- device: {b['ms_per_step']} ms/step, {b['value']} tok/s; roofline {b['roofline']['achieved']} GB/s = "
          f"{b['roofline']['frac']} of the measured {b['roofline']['peak']} GB/s ({b['roofline']['frac_of_8TBs']} of 8 TB/s)")
    print(f"- e2e through `mk_step_tokens` (host token ids in / greedy ids out every step): {b['e2e']['value']} tok/s "
          f"({b['e2e']['ms_per_step']} ms)")
    print(f"- CPU reference arm (`--impl reference`, fp32 oracle, {r['cpu_baseline']['cores']} host threads): "
          f"{r['value']} tok/s ({r['ms_per_step']} ms/step)")
    print("\n## Batch sweep: die-aware (chiplet_m_tile) vs the flat die-unaware megakernel (standard)\n")
    print("| batch | die-aware ms | tok/s | HBM frac (measured peak) | flat ms | die-aware speed-up |\n|---|---|---|---|---|---|")
    for bb in (1, 2, 3, 4, 8, 16, 32, 64):
        try:
            a = J(d, f"b{bb}_m_tile.json")
        except Exception:
            continue
        try:
            f = J(d, f"b{bb}_standard.json")
            fs, sp = f"{f['ms_per_step']}", f"{f['ms_per_step'] / a['ms_per_step']:.2f}x"
        except Exception:
            fs, sp = "-", "-"
        print(f"| {bb} | {a['ms_per_step']} | {a['value']} | {a['roofline']['frac']} | {fs} | {sp} |")
    print("\n## Ablations\n\n| config | B=32 ms | B=64 ms |\n|---|---|---|")
    for tag, name in (("m_tile", "chiplet_m_tile (default)"), ("m_split", "chiplet_m_split"),
                      ("n_major", "chiplet_n_major"), ("m_tile_noks", "whole tiles (no K-split)"),
                      ("m_tile_tm16", "T_M = 16 (cooperative m-tiles)"), ("standard", "flat")):
        v = []
        for bb in (32, 64):
            try:
                v.append(str(J(d, f"b{bb}_{tag}.json")["ms_per_step"]))
            except Exception:
                v.append("-")
        print(f"| {name} | {v[0]} | {v[1]} |")
    for bb in (1, 16):
        try:
            print(f"\nLast-split attention merge (`MK_FUSE_ATTN_REDUCE=1`) at B={bb}: "
                  f"{J(d, f'b{bb}_fused_reduce.json')['ms_per_step']} ms vs {J(d, f'b{bb}_m_tile.json')['ms_per_step']} ms (off).")
        except Exception:
            pass
    print("\n## L2 hit rate / HBM bytes per launch (ncu, one launch after warm-up)\n")
    print("| config | duration ms | L2 hit % | DRAM read GB | DRAM write GB | DRAM % of peak |\n|---|---|---|---|---|---|")
    for p in sorted(glob.glob(os.path.join(d, "l2", "l2_*.csv"))):
        m = {}
        txt = open(p).read()
        for row in csv.reader(io.StringIO("\n".join(l for l in txt.splitlines() if l.startswith('"')))):
            if len(row) > 14 and "megakernel" in row[4]:
                m[row[12]] = (row[13], row[14])
        if not m:
            continue

        def v(k):
            u, x = m.get(k, ("", "nan"))
            return float(x.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        print(f"| {os.path.basename(p)[3:-4]} | {v('gpu__time_duration.sum') / 1e6:.3f} | "
              f"{v('lts__t_sector_hit_rate.pct'):.1f} | {v('dram__bytes_read.sum') / 1e9:.2f} | "
              f"{v('dram__bytes_write.sum') / 1e9:.3f} | {v('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} |")
    print("\n## Tensor parallelism, TP=2 emulated on this one GPU (half the SMs per rank)\n")
    for bb in (1, 16):
        try:
            t = J(d, f"tp2emu_b{bb}.json")
            print(f"- B={bb}: {t['ms_per_step']} ms/step, {t['value']} tok/s; ranks agree on tokens: "
                  f"{t['config']['ranks_agree_on_tokens']}")
        except Exception:
            pass
    print("\nFiles: `b*_*.json` bench lines, `bench_default.json` / `bench_reference.json`, "
          "`ncu_b{1,64}_summary.md` (+ raw page, source page gz), `launches_b1.csv.gz`, `l2/`, `pytest_gpu.log`.")


if __name__ == "__main__":
    main()
