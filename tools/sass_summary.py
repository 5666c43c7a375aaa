"""SASS instruction-class census of every kernel in libmk.so (evidence that
the tcgen05 / TMA / tensor-core paths are what the binary contains).

    python tools/sass_summary.py > profiles/r02/sass_summary.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_15379_b200", "libmk.so")
CLASSES = [
    ("UTCHMMA / UTC*MMA", r"UTC\w*MMA", "tcgen05.mma (5th-gen tensor core)"),
    ("UTCBAR", r"UTCBAR", "tcgen05.commit -> mbarrier"),
    ("LDTM", r"\bLDTM", "tcgen05.ld (TMEM -> registers)"),
    ("UTCATOMSWS / TMEM alloc", r"UTCATOMSWS|UTCHALLOC|UTCALLOC", "tcgen05.alloc / dealloc"),
    ("UTMALDG", r"UTMALDG", "TMA tensor load (cp.async.bulk.tensor)"),
    ("UBLKCP", r"UBLKCP", "TMA bulk copy (cp.async.bulk)"),
    ("UBLKPF / UTMAPF", r"UBLKPF|UTMAPF", "bulk L2 prefetch"),
    ("HMMA", r"\bHMMA", "mma.sync (attention QK^T / PV)"),
    ("LDSM", r"\bLDSM", "ldmatrix"),
    ("SYNCS", r"\bSYNCS", "mbarrier arrive / wait"),
    ("ELECT", r"\bELECT", "elect.sync"),
    ("RED / ATOM (global)", r"\bRED\b|\bREDG|\bATOMG|\bATOM\b", "event counters, K-split signals"),
    ("MEMBAR / FENCE", r"MEMBAR|FENCE", "fences"),
    ("LDG", r"\bLDG", "global loads"),
    ("STG", r"\bSTG", "global stores"),
    ("FFMA", r"\bFFMA", "fp32 FMA (GEMV body)"),
]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else LIB
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    fn = None
    counts = collections.OrderedDict()
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            counts[fn] = collections.Counter()
            continue
        if fn is None or not re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
            continue
        counts[fn]["total"] += 1
        for name, pat, _ in CLASSES:
            if re.search(pat, line):
                counts[fn][name] += 1
    names = [f for f in counts if "megakernel" in f]
    short = {f: re.sub(r".*megakernelILi(\d+)E.*", r"megakernel<\1>", f) for f in names}
    print("# SASS census of libmk.so (`cuobjdump -sass`, sm_100a)\n")
    print("Instances: <0> general CUDA-core graph, <3> general tcgen05 + K-split, "
          "<6> lean batch-1 GEMV, <7> lean all-tcgen05 (mk_create picks per graph).\n")
    print("| class | meaning | " + " | ".join(short[f] for f in names) + " |")
    print("|---|---|" + "---|" * len(names))
    print("| total SASS instructions | | " + " | ".join(str(counts[f]["total"]) for f in names) + " |")
    for name, _, meaning in CLASSES:
        print(f"| {name} | {meaning} | " + " | ".join(str(counts[f][name]) for f in names) + " |")


if __name__ == "__main__":
    main()
