"""Plain torch elementwise kernels on the config-4 pattern at 2^28 fp64
(y += x: 2 reads + 1 write per element, 24 B), CUDA events over 10 launches:
the library ceiling beside the stream region (measurement tool)."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG
n = 1 << 28
x = torch.ones(n, dtype=torch.float64, device="cuda")
y = torch.zeros(n, dtype=torch.float64, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
s = torch.cuda.Stream()


def t(op, reps=10):
    with torch.cuda.stream(s):
        for _ in range(3):
            op()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            op()
        e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
for name, op, b in [("torch_y_add_x", lambda: y.add_(x), 24), ("torch_copy_y_x", lambda: y.copy_(x), 16),
                    ("torch_y_addcmul", lambda: y.add_(x, alpha=2.0), 24),
                    ("stream_region", lambda: RG.run_stream(x, y, [1.0] * 8, sms * 7, 96, stats=False,
                                                            stream=s), 24)]:
    ms = t(op)
    out[name] = round(b * n / ms / 1e6, 1)
print(json.dumps(out))
