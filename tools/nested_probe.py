"""Config-3 kernel for ncu: 1 team x 96 workers, 2000 nested regions
(measurement tool, not product)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
a = torch.zeros(96, dtype=torch.float64, device='cuda')
RG.run_nested(a, 1, 96, 10)
RG.run_nested(a, 1, 96, 2000)
torch.cuda.synchronize()
print("nested probe done")
