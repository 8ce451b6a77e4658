import sys, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
import bench as BN
s = torch.cuda.Stream()
a = torch.zeros(32, dtype=torch.float64, device='cuda')
RG.run_regions(a, 1, 32, 10, stream=s); s.synchronize()
R = 10000
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); RG.run_regions(a, 1, 32, R, stream=s); e1.record(s); e1.synchronize()
    plain = e0.elapsed_time(e1) * 1e6 / R
    dev = BN.device_ms(s, lambda: RG.run_regions(a, 1, 32, R, stream=s)) * 1e6 / R
    print(f"plain {plain:7.1f} ns   device_ms {dev:7.1f} ns")
