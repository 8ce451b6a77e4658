"""Config-3 kernel on the whole GPU (1184 teams x 96 workers, 500 nested
regions) for ncu (measurement tool, not product)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
a = torch.zeros(1184 * 96, dtype=torch.float64, device='cuda')
RG.run_nested(a, 1184, 96, 10)
RG.run_nested(a, 1184, 96, 500)
torch.cuda.synchronize()
print("nested full probe done")
