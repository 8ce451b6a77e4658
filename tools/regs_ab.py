"""A/B of register budgets (OMPDS_LIB_PATH builds with different
OMPDS_GENERIC_LB): config-1 single-team latency and whole-GPU regions/s at
several teams/SM, config-3 per team-region at several teams/SM, config 4
GB/s (measurement tool, not product)."""
import os, statistics, sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG

sms = torch.cuda.get_device_properties(0).multi_processor_count
s = torch.cuda.Stream()


def dms(fn, reps=3):
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000)
        e0.record(); fn(); e1.record(); e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


res = {}
a = torch.zeros(32, dtype=torch.float64, device="cuda")
RG.run_regions(a, 1, 32, 10)
res["cfg1_1team_ns"] = dms(lambda: RG.run_regions(a, 1, 32, 10000)) * 1e6 / 10000
for k in (16, 18, 20, 21):
    t = sms * k
    a2 = torch.zeros(t * 32, dtype=torch.float64, device="cuda")
    RG.run_regions(a2, t, 32, 10)
    ms = dms(lambda: RG.run_regions(a2, t, 32, 2000))
    res[f"cfg1_{k}perSM_Gps"] = t * 2000 / ms / 1e6
for k in (8, 10):
    t = sms * k
    a3 = torch.zeros(t * 96, dtype=torch.float64, device="cuda")
    RG.run_nested(a3, t, 96, 10)
    ms = dms(lambda: RG.run_nested(a3, t, 96, 500, collect=False))
    res[f"cfg3_{k}perSM_ns_per_team_region"] = ms * 1e6 / 500
    res[f"cfg3_{k}perSM_Gps"] = t * 500 / ms / 1e6
a1 = torch.zeros(96, dtype=torch.float64, device="cuda")
RG.run_nested(a1, 1, 96, 10)
res["cfg3_1team_ns"] = dms(lambda: RG.run_nested(a1, 1, 96, 2000, collect=False)) * 1e6 / 2000
n = 1 << 28
x = torch.empty(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
RG.fill_uniform(x, 1); RG.fill_uniform(y, 2)
coef = [k / 8 for k in range(1, 9)]
RG.run_stream(x, y, coef, sms * 7, 96, stats=False)
ms = dms(lambda: [RG.run_stream(x, y, coef, sms * 7, 96, stats=False) for _ in range(20)]) / 20
res["cfg4_GBps"] = 24 * n / ms / 1e6
print(os.environ.get("OMPDS_LIB_PATH", "default"), {k: round(v, 2) for k, v in res.items()})
