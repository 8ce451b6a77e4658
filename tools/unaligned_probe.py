"""Config-4 and config-2 throughput for views that are not 16-byte aligned
(element-wise variants) beside the aligned ones (measurement tool, not
product)."""
import statistics, sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG

sms = torch.cuda.get_device_properties(0).multi_processor_count
coef = [k / 8 for k in range(1, 9)]


def ms_of(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(reps)]; e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps


n = (1 << 28)
bx = torch.empty(n + 2, dtype=torch.float64, device="cuda"); by = torch.empty_like(bx)
RG.fill_uniform(bx, 1); RG.fill_uniform(by, 2)
for label, off in (("aligned", 0), ("offset 1 element", 1)):
    m = n - 2
    x, y = bx[off:off + m], by[off:off + m]
    for teams, w in ((sms * 7, 96), (sms * 4, 224), (sms * 2, 480)):
        ms = ms_of(lambda: RG.run_stream(x, y, coef, teams, w, stats=False))
        print(f"config4 {label:18s} {teams}x{w}: {ms:.3f} ms {24 * m / ms / 1e6:.0f} GB/s")
n2 = 1 << 24
base = torch.zeros(n2 + 2, dtype=torch.float64, device="cuda")
d = torch.arange(256, dtype=torch.float64, device="cuda") * 3 + 1
for label, off in (("aligned", 0), ("offset 1 element", 1)):
    a = base[off:off + n2]
    ms = ms_of(lambda: RG.run_shared_array(a, 296, 480, d_init=d))
    print(f"config2 {label:18s}: {ms * 1e3:.1f} us {16 * n2 / ms / 1e6:.0f} GB/s (L2-warm, back to back)")
