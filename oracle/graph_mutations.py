"""Malformed-graph constructions for validate_graph error-path parity (test
infrastructure).  Each mutation takes a valid toy-layer TaskGraph (from
either builder: only dataclasses.replace and field names are used) and
returns a graph that the reference's validate_graph rejects
(ref taskgraph.py:555-612).  oracle/gen_extra_golden.py records the
reference's messages; tests/test_api_parity.py applies the same mutations
to this package's graphs."""

from dataclasses import replace


def _tasks(g, fn):
    return replace(g, tasks=tuple(fn(list(g.tasks))))


def duplicate_ids(g):
    return _tasks(g, lambda ts: ts + [ts[0]])


def unknown_wait(g):
    def f(ts):
        t = next(t for t in ts if t.wait_events)
        i = ts.index(t)
        ts[i] = replace(t, wait_events=("no.such.event",))
        return ts
    return _tasks(g, f)


def unknown_signal(g):
    def f(ts):
        i = next(i for i, t in enumerate(ts) if t.signal_event)
        ts[i] = replace(ts[i], signal_event="no.such.event")
        return ts
    return _tasks(g, f)


def chiplet_unbound(g):
    def f(ts):
        i = next(i for i, t in enumerate(ts) if t.level.value == "chiplet")
        ts[i] = replace(ts[i], xcd_binding=None)
        return ts
    return _tasks(g, f)


def chiplet_bad_xcd(g):
    def f(ts):
        i = next(i for i, t in enumerate(ts) if t.level.value == "chiplet")
        ts[i] = replace(ts[i], xcd_binding=7)
        return ts
    return _tasks(g, f)


def cu_bound(g):
    def f(ts):
        i = next(i for i, t in enumerate(ts) if t.level.value != "chiplet")
        ts[i] = replace(ts[i], xcd_binding=0)
        return ts
    return _tasks(g, f)


def count_mismatch(g):
    eid = next(iter(g.events))
    ev = g.events[eid]
    ev2 = dict(g.events)
    ev2[eid] = replace(ev, required_count=ev.required_count + 1)
    return replace(g, events=ev2)


def unknown_downstream(g):
    eid = next(e for e, ev in g.events.items() if ev.downstream_tasks)
    ev = g.events[eid]
    ev2 = dict(g.events)
    ev2[eid] = replace(ev, downstream_tasks=tuple(ev.downstream_tasks) + ("no.such.task",))
    return replace(g, events=ev2)


def cycle(g):
    # the first task that signals an event also waits on the event that the
    # first waiter of its own signal signals
    def f(ts):
        src = next(t for t in ts if t.signal_event)
        waiter = next(t for t in ts if src.signal_event in t.wait_events and t.signal_event)
        i = ts.index(src)
        ts[i] = replace(src, wait_events=tuple(src.wait_events) + (waiter.signal_event,))
        return ts
    return _tasks(g, f)


MUTATIONS = {
    "duplicate_ids": duplicate_ids, "unknown_wait": unknown_wait,
    "unknown_signal": unknown_signal, "chiplet_unbound": chiplet_unbound,
    "chiplet_bad_xcd": chiplet_bad_xcd, "cu_bound": cu_bound,
    "count_mismatch": count_mismatch, "unknown_downstream": unknown_downstream,
    "cycle": cycle,
}

# builder argument errors (ref taskgraph.py:371-378)
BUILD_ERRORS = {
    "bad_mode": dict(mode="bogus", batch=1, layers=1),
    "zero_batch": dict(mode="chiplet", batch=0, layers=1),
    "zero_layers": dict(mode="chiplet", batch=1, layers=0),
}
