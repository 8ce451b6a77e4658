"""Per-launch cost of the team kernel with the config-2 geometry (296 teams
x 480 workers) on tiny inputs, queued back to back behind a long spin so the
host is never the bound: kernel with 0 and 1 parallel regions (RegionsProg),
the config-2 and stream regions (measurement tool)."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG
from paper_1711_10413_b200 import _lib as L
import ctypes as C
s = torch.cuda.Stream()
sms = torch.cuda.get_device_properties(0).multi_processor_count
T, W = sms * 2, 480
a = torch.zeros(T * W, dtype=torch.float64, device="cuda")
c = torch.zeros(1 << 14, dtype=torch.float64, device="cuda")
x = torch.ones(1 << 14, dtype=torch.float64, device="cuda")
d = torch.arange(256, dtype=torch.float64, device="cuda")
go2 = RG.prepared_shared_array(c, T, W, d_init=d, stream=s)
out = {}


def regions(n):
    launch = RG.make_launch(T, W, stream=s)
    return lambda: L.lib().ompds_run_regions(C.byref(launch), 1, n, C.c_void_p(a.data_ptr()),
                                             None, None)


for name, op in [("regions_0", regions(0)), ("regions_1", regions(1)), ("regions_4", regions(4)),
                 ("config2", go2),
                 ("stream", lambda: RG.run_stream(x, c, [1.0] * 8, T, W, stats=False, stream=s))]:
    with torch.cuda.stream(s):
        for _ in range(5):
            op()
        torch.cuda._sleep(60_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(200):
            op()
        e1.record(s)
    e1.synchronize()
    out[name + "_us"] = round(e0.elapsed_time(e1) / 200 * 1e3, 2)
print(json.dumps(out))
