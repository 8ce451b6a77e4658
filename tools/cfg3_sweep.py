#!/usr/bin/env python
"""Config 3 on B200: ns per nested region on one team (1 x 96) and
whole-GPU regions/s for a range of 128-thread teams per SM (library at
OMPDS_LIB_PATH; CUDA events, 2000 regions; measurement tool)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1711_10413_b200 import regions as RG  # noqa: E402


def dev_ms(fn, reps=3):
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


sms = torch.cuda.get_device_properties(0).multi_processor_count
R = 2000
out = {}
a = torch.zeros(96, dtype=torch.float64, device="cuda")
out["ns_1team"] = round(dev_ms(lambda: RG.run_nested(a, 1, 96, R, collect=False)) * 1e6 / R, 1)
for per_sm in [int(v) for v in os.environ.get("PER_SM", "8,9,10,12,14,16").split(",")]:
    t = sms * per_sm
    a = torch.zeros(t * 96, dtype=torch.float64, device="cuda")
    ms = dev_ms(lambda: RG.run_nested(a, t, 96, R, collect=False))
    out[per_sm] = round(t * R / (ms * 1e-3) / 1e9, 3)
print(os.path.basename(os.environ.get("OMPDS_LIB_PATH", "default")), json.dumps(out))
