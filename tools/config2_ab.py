"""Config-2 time per launch (L2 evicted before each) for a library build and
a few team geometries (measurement tool, not product)."""
import os, statistics, sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG
n2 = 1 << 24
a = torch.zeros(n2, dtype=torch.float64, device="cuda")
d = torch.arange(256, dtype=torch.float64, device="cuda") * 3 + 1
flush = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
out = []
for k, w in ((2, 480), (4, 224), (7, 96), (8, 96), (1, 992), (3, 480)):
    go = RG.prepared_shared_array(a, 148 * k, w, d_init=d, stream=s)
    go()
    ts = []
    for _ in range(15):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            flush.sum(); torch.cuda._sleep(100_000); e0.record(s); go(); e1.record(s)
        e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    out.append(f"{148*k}x{w}: {16 * n2 / ms / 1e6:6.0f}")
print(f"{os.path.basename(os.environ.get('OMPDS_LIB_PATH', 'default')):16s} " + "  ".join(out), flush=True)
