"""Config-2 kernel at the bench geometry (592 teams x 224 workers, 2^24
doubles, d[256] staged by TMA) for ncu (measurement tool, not product)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG
n = 1 << 24
a = torch.zeros(n, dtype=torch.float64, device="cuda")
d = torch.arange(256, dtype=torch.float64, device="cuda") * 3 + 1
RG.run_shared_array(a, 592, 224, d_init=d)
RG.run_shared_array(a, 592, 224, d_init=d)
torch.cuda.synchronize()
print("config2 probe done")
