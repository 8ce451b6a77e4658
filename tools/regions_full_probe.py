"""Config-1 kernel on the whole GPU (20 teams/SM x 32 workers, 2000 regions)
for ncu (measurement tool, not product)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
t = torch.cuda.get_device_properties(0).multi_processor_count * 20
a = torch.zeros(t * 32, dtype=torch.float64, device='cuda')
RG.run_regions(a, t, 32, 10)
RG.run_regions(a, t, 32, 2000)
torch.cuda.synchronize()
print("regions full probe done")
