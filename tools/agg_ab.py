"""Config-1 (2 int + 2 double captures) latency and whole-GPU regions/s for
A/B of library builds (measurement tool, not product)."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
sms = torch.cuda.get_device_properties(0).multi_processor_count
res = []
for teams, R in ((1, 10000), (sms * 16, 2000), (sms * 20, 2000), (sms * 24, 2000)):
    a = torch.zeros(teams * 32, dtype=torch.float64, device='cuda')
    RG.run_regions(a, teams, 32, 10)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); RG.run_regions(a, teams, 32, R); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
    res.append(f"{teams}t: {ms*1e6/R:6.1f} ns {teams*R/(ms*1e-3)/1e9:5.2f} G/s")
print(f"{os.environ.get('OMPDS_LIB_PATH','default'):28s} " + " | ".join(res))
