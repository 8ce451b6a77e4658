"""Config-3 timing (1 team and 1184 teams) for A/B of library builds
(measurement tool, not product)."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
out = []
for teams in (1, 1184):
    a = torch.zeros(teams * 96, dtype=torch.float64, device='cuda')
    RG.run_nested(a, teams, 96, 10)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); RG.run_nested(a, teams, 96, 2000, collect=False); e1.record(); e1.synchronize()
    out.append(e0.elapsed_time(e1) * 1e6 / 2000)
print(f"{os.environ.get('OMPDS_LIB_PATH', 'default'):32s} 1 team {out[0]:7.1f} ns  1184 teams {out[1]:7.1f} ns")
