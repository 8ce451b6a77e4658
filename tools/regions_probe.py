import sys, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
a = torch.zeros(32, dtype=torch.int32, device='cuda')
RG.run_regions(a, 1, 32, 10)
RG.run_regions(a, 1, 32, 2000)
torch.cuda.synchronize()
print(a[:4].tolist())
