"""Tile schedules of one die's GEMM partition (drop-in for ``chipletsim.traversal``).

The reference decides which worker computes which ``(m, n)`` output tile of
a die's ``[M, K] x [K, N_local]`` slice and in which order
(``/root/reference/pkg/src/chipletsim/traversal.py:125-202``).  The same
assignment rules run on the device inside the persistent kernel's tile loop
(``csrc/mk_sched.cuh`` ``tile_of``), so this module is both the host-side API
and the specification the device loop is tested against.

The reference's line-granular ``AccessStream`` is a cache-simulator artifact
and is not carried over: on B200 the traffic is measured, not simulated.  Its
cache-modifier roles survive as the PTX hints the kernel puts on each stream
(weights ``L2::evict_first`` bulk copies, activations default loads, outputs
plain stores) -- see DESIGN.md.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum


class ScheduleError(ValueError):
    """Bad partition / schedule arguments (ref traversal.py:45)."""


class Traversal(Enum):
    N_MAJOR = "n_major"
    M_MAJOR_WINDOWED = "m_major_windowed"


class Distribution(Enum):
    M_TILE = "m_tile"
    M_SPLIT = "m_split"


def _cdiv(a: int, b: int) -> int:
    return (a + b - 1) // b


@dataclass(frozen=True)
class GemmPartition:
    """One die's slice of a GEMM (ref traversal.py:59-105).

    ``weight_base`` / ``act_base`` / ``out_base`` are the reference's abstract
    byte offsets; the device lowering replaces them with real pointers.
    """

    M: int
    K: int
    N_local: int
    T_M: int
    T_N: int
    T_K: int
    weight_base: int
    act_base: int
    out_base: int
    dtype_bytes: int
    fused_halves: bool = False

    def __post_init__(self):
        for name in ("M", "K", "N_local", "T_M", "T_N", "T_K", "dtype_bytes"):
            if getattr(self, name) <= 0:
                raise ScheduleError(f"nonpositive {name}")

    @property
    def m_tiles(self) -> int:
        return _cdiv(self.M, self.T_M)

    @property
    def n_tiles(self) -> int:
        return _cdiv(self.N_local, self.T_N)

    @property
    def k_chunks(self) -> int:
        return _cdiv(self.K, self.T_K)

    @property
    def weight_bytes(self) -> int:
        return self.dtype_bytes * self.K * self.N_local


@dataclass(frozen=True)
class TileSchedule:
    """Per-worker ordered tile lists plus the concurrency slots."""

    worker_tiles: tuple
    slots: tuple
    traversal: Traversal
    distribution: Distribution
    workers: int


def tile_owner(traversal: Traversal, distribution: Distribution,
               m: int, n: int, m_tiles: int, n_tiles: int,
               workers: int) -> int:
    """Worker that owns tile ``(m, n)`` -- the rule the device loop inverts."""
    if distribution is Distribution.M_SPLIT:
        return n % workers
    if traversal is Traversal.M_MAJOR_WINDOWED:
        return (n * m_tiles + m) % workers
    return (m * n_tiles + n) % workers


def global_order(p_m_tiles: int, p_n_tiles: int, traversal: Traversal,
                 distribution: Distribution, xcd: int):
    """Tiles of the grid in the order the die executes them."""
    if distribution is Distribution.M_SPLIT:
        first = xcd % p_m_tiles
        return [((first + i) % p_m_tiles, n)
                for i in range(p_m_tiles) for n in range(p_n_tiles)]
    if traversal is Traversal.M_MAJOR_WINDOWED:
        return [(idx % p_m_tiles, idx // p_m_tiles)
                for idx in range(p_m_tiles * p_n_tiles)]
    return [(idx // p_n_tiles, idx % p_n_tiles)
            for idx in range(p_m_tiles * p_n_tiles)]


def schedule(p: GemmPartition, workers: int, traversal: Traversal,
             distribution: Distribution, xcd: int = 0, num_xcds: int = 1,
             window: int = 1) -> TileSchedule:
    """Assign ``p``'s tile grid to ``workers`` workers (ref traversal.py:125-202).

    * M_TILE / M_MAJOR_WINDOWED: tiles run down a weight column (all m for one
      n) before the next column; worker ``w`` owns global indices
      ``w, w+W, ...``.  A slot holds whole columns, widened to keep every
      worker busy when a column has fewer tiles than workers.
    * M_TILE / N_MAJOR: tiles run along a batch row; slots of ``W`` tiles.
    * M_SPLIT: column ``n`` always belongs to worker ``n % W``; rows start at
      ``xcd % m_tiles``; slots never cross a row.
    """
    if workers < 1:
        raise ScheduleError("need at least one worker")
    if window < 1:
        raise ScheduleError("window must be at least one column group")
    if not (0 <= xcd < num_xcds):
        raise ScheduleError(f"xcd {xcd} out of range for {num_xcds} XCDs")
    mt, nt = p.m_tiles, p.n_tiles
    order = global_order(mt, nt, traversal, distribution, xcd)

    def own(m, n):
        return tile_owner(traversal, distribution, m, n, mt, nt, workers)

    per_worker = [[] for _ in range(workers)]
    for m, n in order:
        per_worker[own(m, n)].append((m, n))

    if distribution is Distribution.M_SPLIT:
        groups = []
        for r in range(mt):
            row = order[r * nt:(r + 1) * nt]
            groups.extend(row[j:j + workers] for j in range(0, nt, workers))
    else:
        if traversal is Traversal.M_MAJOR_WINDOWED:
            width = mt * max(window, _cdiv(workers, mt))
        else:
            width = workers
        groups = [order[i:i + width] for i in range(0, len(order), width)]
    slots = tuple(tuple((m, n, own(m, n)) for m, n in g) for g in groups)
    return TileSchedule(
        worker_tiles=tuple(tuple(t) for t in per_worker),
        slots=slots,
        traversal=traversal,
        distribution=distribution,
        workers=workers,
    )


def schedule_to_json(s: TileSchedule) -> dict:
    """Stable JSON of a schedule (ref traversal.py:342-354)."""
    return {
        "schema_version": 1,
        "traversal": s.traversal.value,
        "distribution": s.distribution.value,
        "workers": [[list(t) for t in tiles] for tiles in s.worker_tiles],
        "slots": [[list(e) for e in slot] for slot in s.slots],
    }
