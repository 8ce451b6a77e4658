"""Fixed cost per launch of the config-2 region (TMA staging of d[] +
protocol) against the stream region and a torch elementwise kernel on a
tiny array, same 296 x 480 team geometry: per-launch time of 200 queued
launches (measurement tool)."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG
s = torch.cuda.Stream()
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = {}
for n in (1 << 14, 1 << 20):
    a = torch.zeros(n, dtype=torch.float64, device="cuda")
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    d = torch.arange(256, dtype=torch.float64, device="cuda")
    go = RG.prepared_shared_array(a, sms * 2, 480, d_init=d, stream=s)
    go_o = RG.prepared_shared_array(a, sms * 2, 480, d_init=d, stream=s, depot_capacity=0)
    for name, op in [("config2", go), ("config2_depot_on_chain", go_o),
                     ("stream_296x480", lambda: RG.run_stream(x, a, [1.0] * 8, sms * 2, 480,
                                                              stats=False, stream=s)),
                     ("torch_add_", lambda: a.add_(1.0))]:
        with torch.cuda.stream(s):
            for _ in range(5):
                op()
            torch.cuda._sleep(40_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(200):
                op()
            e1.record(s)
        e1.synchronize()
        out[f"{name}_n{n}_us"] = round(e0.elapsed_time(e1) / 200 * 1e3, 2)
print(json.dumps(out, indent=1))
