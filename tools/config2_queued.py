"""Config-2 GB/s per team geometry for the library at OMPDS_LIB_PATH:
single launch after an L2-evicting read (event-bracketed) and queued
steady state (K x [evict; region] - K x [evict]), which includes the
write-back of the dirty lines a launch leaves in L2 (measurement tool)."""
import os, statistics, sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG
n2 = 1 << 24
a = torch.zeros(n2, dtype=torch.float64, device="cuda")
d = torch.arange(256, dtype=torch.float64, device="cuda") * 3 + 1
flush = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
K = 20
geoms = [tuple(int(v) for v in g.split("x")) for g in os.environ.get("GEOMS", "2x480,3x480,4x480,4x224,6x224,8x224").split(",")]
out = []
for k, w in geoms:
    go = RG.prepared_shared_array(a, 148 * k, w, d_init=d, stream=s)
    go()

    def queued(with_region):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            torch.cuda._sleep(200_000)
            e0.record(s)
            for _ in range(K):
                flush.sum()
                if with_region:
                    go()
            e1.record(s)
        e1.synchronize()
        return e0.elapsed_time(e1)
    queued(True)
    both = statistics.median(queued(True) for _ in range(3))
    alone = statistics.median(queued(False) for _ in range(3))
    ms = (both - alone) / K
    out.append(f"{148*k}x{w}:{16 * n2 / ms / 1e6:5.0f}")
print(f"{os.path.basename(os.environ.get('OMPDS_LIB_PATH', 'default')):16s} " + " ".join(out), flush=True)
