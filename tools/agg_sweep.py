"""Aggregate parallel regions/s of the config-1 protocol vs team geometry
(measurement tool, not product; CUDA events on one B200)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
sms = torch.cuda.get_device_properties(0).multi_processor_count
for w in (32, 64, 96):
    for k in (4, 8, 16, 24, 32):
        teams = sms * k
        R = 2000
        a = torch.zeros(teams * w, dtype=torch.int32, device='cuda')
        try:
            RG.run_regions(a, teams, w, 10)
        except Exception as e:
            print(w, k, 'fail', e); continue
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); RG.run_regions(a, teams, w, R); e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"W={w:3d} teams/SM={k:2d}: {teams*R/(ms*1e-3)/1e9:6.2f} G regions/s  {ms*1e6/R:7.1f} ns/region/team")
