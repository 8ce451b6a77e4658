import sys, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
for R in (3, 10, 255, 256, 257, 300, 2000):
    a = torch.zeros(96, dtype=torch.float64, device='cuda')
    _, st = RG.run_nested(a, 1, 96, R)
    print(R, st[0][0])
