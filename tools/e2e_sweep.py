"""e2e (host buffers through the C ABI) vs library build: chunk-size sweep
(measurement tool, not product)."""
import os, sys, time, torch
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
n = 1 << 28
COEF = [k / 8 for k in range(1, 9)]
xh = torch.empty(n, dtype=torch.float64).pin_memory()
yh = torch.empty(n, dtype=torch.float64).pin_memory()
xd = torch.empty(n, dtype=torch.float64, device='cuda')
yd = torch.empty(n, dtype=torch.float64, device='cuda')
s = torch.cuda.Stream()
RG.run_stream_host(xh, yh, COEF, 1184, 96, xd, yd, stream=s)
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); RG.run_stream_host(xh, yh, COEF, 1184, 96, xd, yd, stream=s); e1.record(s); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
print(f"{os.environ.get('OMPDS_LIB_PATH','default'):40s} {24*n/(ms*1e-3)/1e9:7.2f} GB/s  {ms:7.2f} ms")
# host link: each direction alone, then both at once (2 GiB each way)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
def timed(pairs):
    evs = []
    for st, dst, src in pairs:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st); dst.copy_(src, non_blocking=True); e1.record(st)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return [8 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9 for e0, e1 in evs]
timed([(sa, xd, xh)])
print("h2d alone %.1f GB/s" % timed([(sa, xd, xh)])[0])
print("d2h alone %.1f GB/s" % timed([(sb, yh, yd)])[0])
print("h2d + d2h concurrently: %.1f / %.1f GB/s" % tuple(timed([(sa, xd, xh), (sb, yh, yd)])))
