"""Config-4 GB/s of the product kernel over team geometries (measurement
tool, not a bench value): teams = 148 x k, W workers (+ the master warp)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG
COEF = [k / 8 for k in range(1, 9)]
n = 1 << 28
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
RG.fill_uniform(x, 0x5eed01ab)
RG.fill_uniform(y, 0x5eed01ac)
res = []
for w in (64, 96, 128, 160, 224):
    for k in (6, 7, 8, 9, 10, 12):
        thr = (w + 31) // 32 * 32 + 32
        if k * thr > 2048:
            continue
        teams = 148 * k
        try:
            for _ in range(3):
                RG.run_stream(x, y, COEF, teams, w, stats=False)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(40):
                RG.run_stream(x, y, COEF, teams, w, stats=False)
            e1.record(); e1.synchronize()
            gbs = 24 * n * 40 / (e0.elapsed_time(e1) * 1e-3) / 1e9
        except Exception as e:
            gbs = float('nan')
        res.append((gbs, w, k))
        print(f"W={w:4d} teams/SM={k:2d} ({teams} teams): {gbs:7.1f} GB/s", flush=True)
print("best", max(r for r in res if r[0] == r[0]))
