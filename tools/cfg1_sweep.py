#!/usr/bin/env python
"""Config 1 on B200: ns per region on one team (int / double captures) and
whole-GPU regions/s for a range of teams per SM (one 64-thread team = W 32
workers + the master warp).  CUDA events; 1 s idle before the single-team
runs so the SM clock is at its maximum."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_10413_b200 import regions as RG  # noqa: E402


def dev_ms(fn, reps=5):
    ts = []
    for i in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    out = {}
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    time.sleep(1.0)
    R = 10000
    for dt in (torch.int32, torch.float64):
        a = torch.zeros(32, dtype=dt, device="cuda")
        out[f"ns_per_region_1team_{dt}"] = dev_ms(lambda: RG.run_regions(a, 1, 32, R)) * 1e6 / R
    R2 = 2000
    agg = {}
    for per_sm in [int(x) for x in os.environ.get("PER_SM", "16,18,20,21,22,23,24,25,26,28,30,32").split(",")]:
        teams = sms * per_sm
        a = torch.zeros(teams * 32, dtype=torch.float64, device="cuda")
        ms = dev_ms(lambda: RG.run_regions(a, teams, 32, R2), reps=7)
        agg[per_sm] = teams * R2 / (ms * 1e-3)
    out["regions_per_s_by_teams_per_sm"] = agg
    print(json.dumps(out, indent=1))
    if len(sys.argv) > 1:
        json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
