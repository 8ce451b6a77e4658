"""Tiny config-2 launch (2^14 elements, 296 x 480 teams) for ncu: the
region's fixed per-launch cost (measurement tool)."""
import sys, torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG
sms = torch.cuda.get_device_properties(0).multi_processor_count
a = torch.zeros(1 << 14, dtype=torch.float64, device="cuda")
d = torch.arange(256, dtype=torch.float64, device="cuda")
go = RG.prepared_shared_array(a, sms * 2, 480, d_init=d)
for _ in range(5):
    go()
torch.cuda.synchronize()
