"""Is config 2's gap to a same-size copy the in-place read-modify-write?
Queued steady state (K x [evict; op] - K x [evict], the bench's method) for
config 2, torch copy_ (two buffers), torch in-place add_ of a scalar and of a
256-periodic tensor (the same RMW pattern as config 2), and our stream
region at 2^24 (measurement tool)."""
import json, statistics, sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG

n2 = 1 << 24
dev = "cuda"
a = torch.zeros(n2, dtype=torch.float64, device=dev)
src = torch.ones(n2, dtype=torch.float64, device=dev)
d = torch.arange(256, dtype=torch.float64, device=dev) * 3 + 1
dper = d.repeat(n2 // 256)
flush = torch.ones(64 << 20, dtype=torch.int32, device=dev)
s = torch.cuda.Stream()
K = 20
sms = torch.cuda.get_device_properties(0).multi_processor_count


def queued(op):
    def run(with_op):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            torch.cuda._sleep(200_000)
            e0.record(s)
            for _ in range(K):
                flush.sum()
                if with_op:
                    op()
            e1.record(s)
        e1.synchronize()
        return e0.elapsed_time(e1)
    run(True)
    both = statistics.median(run(True) for _ in range(5))
    alone = statistics.median(run(False) for _ in range(5))
    return (both - alone) / K


go2 = RG.prepared_shared_array(a, sms * 2, 480, d_init=d, stream=s)
x = torch.ones(n2, dtype=torch.float64, device=dev)
y = torch.zeros(n2, dtype=torch.float64, device=dev)
out = {}
with torch.cuda.stream(s):
    for name, op, byts in [
        ("config2_region", go2, 16 * n2),
        ("torch_copy", lambda: a.copy_(src), 16 * n2),
        ("torch_add_scalar_inplace", lambda: a.add_(1.0), 16 * n2),
        ("torch_add_periodic_inplace", lambda: a.add_(dper), 24 * n2),
        ("stream_region_2^24", lambda: RG.run_stream(x, y, [1.0] * 8, sms * 7, 96, stats=False, stream=s), 24 * n2),
    ]:
        ms = queued(op)
        out[name] = {"us": round(ms * 1e3, 2), "GBps": round(byts / ms / 1e6, 1)}
print(json.dumps(out, indent=1))

# config 4 at the bench size (2^28, inputs > L2): 10 launches, CUDA events
if "--no-big" not in sys.argv:
    del x, y, a, src, dper
    n4 = 1 << 28
    x4 = torch.ones(n4, dtype=torch.float64, device=dev)
    y4 = torch.zeros(n4, dtype=torch.float64, device=dev)
    with torch.cuda.stream(s):
        for _ in range(3):
            RG.run_stream(x4, y4, [1.0] * 8, sms * 7, 96, stats=False, stream=s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            RG.run_stream(x4, y4, [1.0] * 8, sms * 7, 96, stats=False, stream=s)
        e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    out["stream_region_2^28"] = {"us": round(ms * 1e3, 2), "GBps": round(24 * n4 / ms / 1e6, 1)}
import os
print(os.path.basename(os.environ.get("OMPDS_LIB_PATH", "default")),
      json.dumps({k: v["GBps"] for k, v in out.items()}))
