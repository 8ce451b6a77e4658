"""Chrome/Perfetto trace of the runtime's event log.

The reference traces its simulator instruction by instruction
(`SimOptions::Trace`, proj/src/Simulator.cpp:629-636) and keeps a per-team
`RuntimeEvent` log (proj/include/omplab/DeviceRuntime.h:64-79).  On the GPU
the event log is the trace: every init / prepare / fetch / retire / free /
deinit carries the %globaltimer time it was logged at
(`ompds_event.t_ns`, `Outputs.team_events(times=True)`).  This module turns
those logs into the Trace Event Format (chrome://tracing, ui.perfetto.dev):
one process per team, the master and the worker fetch/retire pairs as
spans, everything else as instants.
"""
from __future__ import annotations

import json
from typing import Dict, List, Sequence


def chrome_trace(team_events: Sequence[Sequence[tuple]], first_team: int = 0) -> Dict:
    """`team_events`: per team, (kind, fn, nargs, bytes, t_ns) tuples in log
    order (`Outputs.team_events(times=True)`).  Returns the trace dict.

    Per team: a "master" track with one span per parallel region (its
    prepare up to the region's last retire or list free) and a "workers"
    track with fetch-to-retire spans (the log records one fetch and one
    retire per participating worker thread but no thread id, so spans pair
    them in log order).  Times are microseconds from the earliest event of
    the launch."""
    times = [e[4] for evs in team_events for e in evs if len(e) > 4]
    if len(times) != sum(len(evs) for evs in team_events):
        raise ValueError("events need device times: team_events(times=True)")
    t0 = min(times) if times else 0
    us = lambda t: (t - t0) / 1e3  # noqa: E731
    out: List[Dict] = []
    for k, evs in enumerate(team_events):
        pid = first_team + k
        out.append({"ph": "M", "name": "process_name", "pid": pid,
                    "args": {"name": f"team {pid}"}})
        for tid, name in ((0, "master"), (1, "workers")):
            out.append({"ph": "M", "name": "thread_name", "pid": pid, "tid": tid,
                        "args": {"name": name}})
        state = {"region": None, "end": None}
        fetches: List[tuple] = []

        def close_region():
            if state["region"] is not None:
                tp, f, na, pk, nb = state["region"]
                end = state["end"] if state["end"] is not None else tp
                out.append({"ph": "X", "name": f"parallel {f}", "pid": pid, "tid": 0,
                            "ts": us(tp), "dur": max(us(end) - us(tp), 0.0),
                            "args": {"nargs": na, "list": pk.split("_")[1],
                                     "list_bytes": nb}})
            state["region"], state["end"] = None, None

        for kind, fn, nargs, nbytes, t in evs:
            if kind in ("prepare_prealloc", "prepare_dynamic"):
                close_region()
                state["region"] = (t, fn, nargs, kind, nbytes)
            elif kind == "fetch":
                fetches.append((t, fn))
            elif kind in ("retire", "dynamic_free"):
                state["end"] = t if state["end"] is None else max(state["end"], t)
                if kind == "retire" and fetches:
                    tf, f = fetches.pop(0)
                    out.append({"ph": "X", "name": f"region {f}", "pid": pid, "tid": 1,
                                "ts": us(tf), "dur": max(us(t) - us(tf), 0.0)})
                if kind == "dynamic_free":
                    out.append({"ph": "i", "s": "t", "name": kind, "pid": pid, "tid": 1,
                                "ts": us(t), "args": {"bytes": nbytes}})
            else:  # init, deinit
                close_region()
                out.append({"ph": "i", "s": "t", "name": kind, "pid": pid, "tid": 0,
                            "ts": us(t), "args": {"fn": fn, "nargs": nargs, "bytes": nbytes}})
        close_region()
    return {"traceEvents": out, "displayTimeUnit": "ns"}


def write_chrome_trace(path: str, team_events: Sequence[Sequence[tuple]],
                       first_team: int = 0) -> None:
    with open(path, "w") as f:
        json.dump(chrome_trace(team_events, first_team), f)
