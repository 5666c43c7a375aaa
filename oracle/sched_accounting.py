"""Restatement of the reference simulator's sync accounting -- TEST INFRASTRUCTURE.

The reference runtime (``/root/reference/pkg/src/chipletsim/runtime.py``)
counts, per executed graph:

* ``dispatches``: one per task -- a chiplet task is broadcast to all workers
  of its die but dispatched once (runtime.py:378-394), a CU / wavefront task
  goes to one worker (runtime.py:395-417);
* ``local_atomics``: every worker of the die increments the die-local counter
  when a chiplet task completes (runtime.py:438-447) -> ``workers_per_xcd``
  per chiplet task;
* ``fences`` and the chiplet part of ``global_atomics``: only the last of
  those increments pays one fence + one global atomic (runtime.py:448-451);
* the CU part of ``global_atomics``: one per completing CU / wavefront task
  with a signal event (runtime.py:469-472).

This module re-derives those counts from a TaskGraph alone (the cache model
and logical steps are not needed for them).  ``tests/test_oracle_sched.py``
pins it against ``tests/golden/sim_counters.json`` produced by the reference's
own ``simulate``; the device counters (``mk_counters``) are then checked
against this restatement in ``tests/test_gpu_megakernel.py``.
"""

from __future__ import annotations


def expected_counters(g, workers_per_xcd: int) -> dict:
    n_chiplet = sum(1 for t in g.tasks if t.level.value == "chiplet")
    n_other = sum(1 for t in g.tasks
                  if t.level.value != "chiplet" and t.signal_event is not None)
    return {
        "dispatches": len(g.tasks),
        "fences": n_chiplet,
        "local_atomics": n_chiplet * workers_per_xcd,
        "global_atomics": n_chiplet + n_other,
    }


def dispatch_partition(g, num_xcds: int):
    """Per-die ready lists in the reference's enqueue order
    (runtime.py:301-307): chiplet tasks to their die, CU/wavefront tasks
    round-robin over dies in graph (= topological) order."""
    lists = [[] for _ in range(num_xcds)]
    rr = 0
    for t in g.tasks:
        if t.level.value == "chiplet":
            lists[t.xcd_binding].append(t.id)
        else:
            lists[rr % num_xcds].append(t.id)
            rr += 1
    return lists
