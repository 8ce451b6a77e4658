"""Config-4 GB/s of a library build (OMPDS_LIB_PATH) at a few team
geometries (measurement tool, not a bench value)."""
import os, sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG
COEF = [k / 8 for k in range(1, 9)]
n = 1 << 28
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
RG.fill_uniform(x, 0x5eed01ab)
RG.fill_uniform(y, 0x5eed01ac)
out = []
for k, w in [tuple(map(int, g.split(","))) for g in os.environ.get("GEOMS", "6,96 7,96 8,96 6,128 8,64 12,64").split()]:
    teams = 148 * k
    for _ in range(3):
        RG.run_stream(x, y, COEF, teams, w, stats=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(40):
        RG.run_stream(x, y, COEF, teams, w, stats=False)
    e1.record(); e1.synchronize()
    out.append(f"{teams}x{w}: {24 * n * 40 / (e0.elapsed_time(e1) * 1e-3) / 1e9:6.0f}")
print(f"{os.path.basename(os.environ.get('OMPDS_LIB_PATH', 'default')):16s} " + "  ".join(out), flush=True)
