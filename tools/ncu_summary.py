"""Summarise an ncu report (raw page) into markdown: duration, DRAM bytes and
throughput, L2 hit rate, tensor-pipe activity, top stall reasons.

    python tools/ncu_summary.py <report.ncu-rep | raw.csv> "<title>" > profiles/rNN/x.md

(a raw.csv is the `ncu -i rep --page raw --csv` export of the report)
"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum.per_second", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_lookup_hit.sum", "lts__t_sectors_srcunit_tex_lookup_miss.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    if rep.endswith(".csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"# ncu summary: {title}", "", f"report: `{rep}`", "",
           "| metric | unit | value |", "|---|---|---|"]
    for r in rows[2:3]:
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                out.append(f"| {w} | {units[i]} | {r[i]} |")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        out += ["", "| stall reason (all warps incl. spinning roles) | share |", "|---|---|"]
        out += [f"| {h} | {100 * v / tot:.1f}% |" for v, h in sorted(stalls, reverse=True)[:8]]
    print("\n".join(out))


if __name__ == "__main__":
    main()
