"""Config-1 kernel (1 team x 32, int+double captures) with 200k regions for
ncu source-level sampling (measurement tool, not product)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
a = torch.zeros(32, dtype=torch.float64, device='cuda')
RG.run_regions(a, 1, 32, 10)
RG.run_regions(a, 1, 32, 200000)
torch.cuda.synchronize()
print("done")
