"""Config-3 whole-GPU time per region vs the number of regions, twice in a
row (measurement tool, not product)."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
for rep in range(2):
    for R in (100, 500, 1000, 2000, 4000):
        a = torch.zeros(1184 * 96, dtype=torch.float64, device='cuda')
        RG.run_nested(a, 1184, 96, 10)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); RG.run_nested(a, 1184, 96, R, collect=False); e1.record(); e1.synchronize()
        print(rep, R, round(e0.elapsed_time(e1) * 1e6 / R, 1), "ns/region", flush=True)
