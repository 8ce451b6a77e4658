"""Config 4 at 2^28: GB/s by team geometry for the library at OMPDS_LIB_PATH
(CUDA events over 10 launches; inputs larger than L2; measurement tool)."""
import json, os, sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG
n = 1 << 28
x = torch.ones(n, dtype=torch.float64, device="cuda")
y = torch.zeros(n, dtype=torch.float64, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
s = torch.cuda.Stream()
out = {}
for per_sm, w in [(7, 96), (8, 96), (9, 96), (5, 160), (4, 224)]:
    t = sms * per_sm
    op = lambda: RG.run_stream(x, y, [1.0] * 8, t, w, stats=False, stream=s)
    with torch.cuda.stream(s):
        for _ in range(3):
            op()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            op()
        e1.record(s)
    e1.synchronize()
    out[f"{t}x{w}"] = round(24 * n / (e0.elapsed_time(e1) / 10) / 1e6, 1)
print(os.path.basename(os.environ.get("OMPDS_LIB_PATH", "default")), json.dumps(out))
