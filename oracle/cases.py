"""Case lists shared by the golden generator and the parity tests.

Test infrastructure only (see oracle/README.md).  Tile specs use the op-kind
string values as keys so the same dict resolves against either package's
``OpKind`` enum.
"""

from __future__ import annotations

import itertools

B200_MACHINE_JSON = {
    "num_xcds": 2,
    "cus_per_xcd": 74,
    "workers_per_xcd": 73,
    "l2_capacity_bytes": 63 * (1 << 20),
    "l2_line_bytes": 128,
    "llc_capacity_bytes": 1 << 20,
    "hbm_bandwidth_bytes_per_s": 8.0e12,
    "l2_bandwidth_bytes_per_s": 2.0e13,
    "peak_flops": 2.25e15,
    "scheduler_mode": "dedicated",
}

_LIN = ("qkv_proj", "o_proj_residual", "gate_up_silu", "down_proj_residual")

TILE_SPECS = {
    "default": None,
    # the reference tests' TOY_TILES (test_taskgraph.py:25-27)
    "toy": dict({k: (16, 16, 64) for k in _LIN}, silu_chunk=16),
    # B200 CUDA-core GEMV tiles: 8 weight rows x 1024-wide K chunks
    "b200_gemv": dict({k: (16, 8, 1024) for k in _LIN}, silu_chunk=128),
    # B200 tcgen05 tiles: 128 weight rows (UMMA M) x 64-wide K chunks
    "b200_umma": dict({k: (16, 128, 64) for k in _LIN}, silu_chunk=128),
    "b200_umma_m64": dict({k: (64, 128, 64) for k in _LIN}, silu_chunk=128),
    "fit": "fit",
}


def tiles_for(spec):
    return TILE_SPECS[spec]


def _graph_cases():
    out = []
    # reference presets, reference tiles
    for mode, b in itertools.product(("standard", "chiplet"), (1, 16, 32, 33)):
        out.append(dict(machine="mi350", model="qwen3-8b", mode=mode,
                        batch=b, layers=1, tiles="default"))
    for mode, b in itertools.product(("standard", "chiplet"), (1, 4, 32)):
        out.append(dict(machine="toy", model="toy", mode=mode, batch=b,
                        layers=2, tiles="toy", full=True))
        out.append(dict(machine="toy", model="toy", mode=mode, batch=b,
                        layers=2, tiles="fit", full=True))
    # the B200 machine at the bench configs
    for mode, b in itertools.product(("standard", "chiplet"),
                                     (1, 2, 4, 8, 16, 32, 64)):
        out.append(dict(machine="b200", model="qwen3-8b", mode=mode,
                        batch=b, layers=1, tiles="b200_gemv"))
        out.append(dict(machine="b200", model="qwen3-8b", mode=mode,
                        batch=b, layers=1, tiles="b200_umma"))
    for mode in ("standard", "chiplet"):
        for b in (1, 64):
            out.append(dict(machine="b200", model="qwen3-8b", mode=mode,
                            batch=b, layers=36, tiles="b200_gemv"))
        out.append(dict(machine="b200", model="qwen3-8b", mode=mode,
                        batch=64, layers=36, tiles="b200_umma_m64"))
        out.append(dict(machine="b200", model="qwen3-8b", mode=mode,
                        batch=1, layers=36, tiles="default"))
        out.append(dict(machine="b200", model="toy", mode=mode, batch=2,
                        layers=2, tiles="fit", full=True))
    return out


GRAPH_CASES = _graph_cases()


def _schedule_cases():
    out = []
    for (mt, nt), w, trav, dist, (xcd, nx), win in itertools.product(
            [(1, 6), (2, 6), (4, 6), (3, 5), (4, 13), (2, 48), (4, 384),
             (1, 384)],
            [1, 3, 4, 73],
            ["m_major_windowed", "n_major"],
            ["m_tile", "m_split"],
            [(0, 1), (1, 2), (0, 2)],
            [1, 2]):
        out.append(dict(m_tiles=mt, n_tiles=nt, workers=w, traversal=trav,
                        distribution=dist, xcd=xcd, num_xcds=nx, window=win))
    return out


SCHEDULE_CASES = _schedule_cases()

SIM_CASES = [
    dict(kind="gemm", machine="mi350", shape=[1, 512, 3968],
         tiles=[16, 16, 256], mode="chiplet", traversal="m_major_windowed",
         distribution="m_tile"),
    dict(kind="gemm", machine="mi350", shape=[1, 512, 3968],
         tiles=[16, 16, 256], mode="standard", traversal="m_major_windowed",
         distribution="m_tile"),
    dict(kind="gemm", machine="b200", shape=[16, 1024, 2048],
         tiles=[16, 8, 256], mode="chiplet", traversal="m_major_windowed",
         distribution="m_tile"),
    dict(kind="layer", machine="toy", model="toy", mode="chiplet", batch=1,
         layers=1, tiles="toy", traversal="m_major_windowed",
         distribution="m_tile", log=True),
    dict(kind="layer", machine="toy", model="toy", mode="chiplet", batch=4,
         layers=2, tiles="toy", traversal="m_major_windowed",
         distribution="m_tile", log=True),
    dict(kind="layer", machine="toy", model="toy", mode="standard", batch=2,
         layers=1, tiles="toy", traversal="m_major_windowed",
         distribution="m_tile", log=True),
    dict(kind="layer", machine="toy", model="toy", mode="chiplet", batch=32,
         layers=1, tiles="toy", traversal="m_major_windowed",
         distribution="m_split"),
    dict(kind="layer", machine="b200", model="toy", mode="chiplet", batch=2,
         layers=2, tiles="fit", traversal="m_major_windowed",
         distribution="m_tile", log=True),
    dict(kind="layer", machine="b200", model="toy", mode="standard", batch=2,
         layers=2, tiles="fit", traversal="m_major_windowed",
         distribution="m_tile"),
]
