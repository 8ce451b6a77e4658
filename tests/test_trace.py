"""Chrome/Perfetto export of the runtime event log (paper_1711_10413_b200/trace.py):
structure on a synthetic log (CPU) and on a real launch (GPU)."""
import json

import pytest

from paper_1711_10413_b200 import trace as TR


def _log(t0, regions, workers, dynamic=False):
    ev, t = [("init", -1, 0, 0, t0)], t0
    for r in range(regions):
        t += 100
        ev.append(("prepare_dynamic" if dynamic else "prepare_prealloc", r, 4, 32 if dynamic else 0, t))
        for w in range(workers):
            t += 10
            ev.append(("fetch", r, 4, 0, t))
        for w in range(workers):
            t += 10
            ev.append(("retire", r, 0, 0, t))
        if dynamic:
            t += 5
            ev.append(("dynamic_free", -1, 0, 32, t))
    ev.append(("deinit", -1, 0, 0, t + 50))
    return ev


def test_chrome_trace_structure_from_a_synthetic_log():
    logs = [_log(1000, 3, 2), _log(1500, 2, 3, dynamic=True)]
    tr = TR.chrome_trace(logs, first_team=4)
    ev = tr["traceEvents"]
    names = {e["args"]["name"] for e in ev if e["name"] == "process_name"}
    assert names == {"team 4", "team 5"}
    spans = [e for e in ev if e["ph"] == "X"]
    # master spans: one per region, from prepare to the last retire / free
    master = [e for e in spans if e["tid"] == 0]
    assert [(e["pid"], e["name"]) for e in master] == [
        (4, "parallel 0"), (4, "parallel 1"), (4, "parallel 2"),
        (5, "parallel 0"), (5, "parallel 1")]
    assert master[0]["ts"] == 0.0 + 0.1 and master[0]["dur"] == pytest.approx(0.04)
    assert master[3]["args"] == {"nargs": 4, "list": "dynamic", "list_bytes": 32}
    # worker spans: one per fetch/retire pair, never negative
    workers = [e for e in spans if e["tid"] == 1]
    assert len(workers) == 3 * 2 + 2 * 3 and all(e["dur"] >= 0 for e in workers)
    inst = [e["name"] for e in ev if e["ph"] == "i"]
    assert inst.count("init") == 2 and inst.count("deinit") == 2 and inst.count("dynamic_free") == 2
    json.dumps(tr)


def test_chrome_trace_needs_device_times():
    with pytest.raises(ValueError):
        TR.chrome_trace([[("init", -1, 0, 0)]])


@pytest.mark.gpu
def test_chrome_trace_of_a_real_launch(tmp_path):
    import torch
    from paper_1711_10413_b200 import regions as RG
    teams, workers, regions = 3, 40, 4
    a = torch.zeros(teams * workers, dtype=torch.int32, device="cuda")
    out = RG.run_regions(a, teams, workers, regions, max_events=1024, prealloc_entries=2)
    path = tmp_path / "trace.json"
    TR.write_chrome_trace(str(path), out.team_events(times=True))
    tr = json.loads(path.read_text())
    spans = [e for e in tr["traceEvents"] if e["ph"] == "X"]
    assert sum(1 for e in spans if e["tid"] == 0) == teams * regions
    assert sum(1 for e in spans if e["tid"] == 1) == teams * regions * workers
    assert all(e["dur"] >= 0 and e["ts"] >= 0 for e in spans)
    master = [e for e in spans if e["tid"] == 0]
    assert all(e["args"]["list"] == "dynamic" for e in master)  # 4 captures > 2-entry window
