"""Config-3 whole-GPU nested regions/s over team geometries (measurement
tool, not product)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
sms = torch.cuda.get_device_properties(0).multi_processor_count
for w in (32, 64, 96, 224):
    for k in (4, 8, 12, 16):
        teams = sms * k
        thr = (w + 31) // 32 * 32 + 32
        if k * thr > 2048:
            continue
        a = torch.zeros(teams * w, dtype=torch.float64, device='cuda')
        RG.run_nested(a, teams, w, 10)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); RG.run_nested(a, teams, w, 1000, collect=False); e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"W={w:3d} teams/SM={k:2d}: {teams * 1000 / (ms * 1e-3) / 1e9:5.2f} G nested regions/s "
              f"({ms * 1e6 / 1000:7.1f} ns per team-region)", flush=True)
