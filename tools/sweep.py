#!/usr/bin/env python
"""Tuning sweep on one GPU (not a bench value): config-4 GB/s over team
geometries, and config-1 region latency / aggregate regions/s."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG  # noqa: E402

COEF = [k / 8 for k in range(1, 9)]


def time_it(fn, reps):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def config2():
    n2 = 1 << 24
    a = torch.zeros(n2, dtype=torch.float64, device="cuda")
    d = torch.arange(256, dtype=torch.float64, device="cuda") * 3 + 1
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for w, per_sm in [(96, 32), (96, 8), (96, 4), (224, 4), (480, 2), (992, 1), (992, 2),
                      (224, 8)]:
        teams = 148 * per_sm
        ts = []
        for _ in range(8):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            RG.run_shared_array(a, teams, w, d_init=d, stats=False) if False else \
                RG.run_shared_array(a, teams, w, d_init=d)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        print({"config2_workers": w, "teams": teams, "ms": round(ms, 4),
               "GBps": round(16 * n2 / ms / 1e6, 1)}, flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "config2":
        return config2()
    out = {"stream": [], "regions": []}
    n = 1 << 28
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    RG.fill_uniform(x, 1)
    RG.fill_uniform(y, 2)
    geoms = [(992, 2), (96, 16), (96, 8), (96, 12), (96, 24), (96, 32), (96, 48), (64, 16),
             (64, 32), (32, 32), (160, 12), (224, 6), (224, 8), (224, 16), (128, 16), (480, 4)]
    if len(sys.argv) > 1 and sys.argv[1] == "quick":
        geoms = geoms[:3]
    if len(sys.argv) > 1 and sys.argv[1] == "regions":
        geoms = []
    for w, per_sm in geoms:
        teams = 148 * per_sm
        ms = time_it(lambda: RG.run_stream(x, y, COEF, teams, w, stats=False), 30)
        out["stream"].append({"workers": w, "teams": teams, "ms": round(ms, 4),
                              "GBps": round(24 * n / ms / 1e6, 1)})
        print(out["stream"][-1], flush=True)
    del x, y
    R = 10000
    for teams, w in [(1, 32), (1, 64), (1, 992), (148, 32), (296, 32), (592, 32), (1184, 32),
                     (148, 96)]:
        a = torch.zeros(teams * w, dtype=torch.int32, device="cuda")
        ms = time_it(lambda: RG.run_regions(a, teams, w, R), 3)
        out["regions"].append({"teams": teams, "workers": w, "ns_per_region": round(ms * 1e6 / R, 1),
                               "aggregate_regions_per_s": round(teams * R / ms * 1e3, 0)})
        print(out["regions"][-1], flush=True)
    json.dump(out, open("gpurun_out/sweep.json", "w"), indent=1)


if __name__ == "__main__":
    main()
