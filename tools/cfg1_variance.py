"""Config-1 single-team region time across fresh allocations of a[] and
across launches with the same a[] (measurement tool, not product): does the
run-to-run spread follow the array's address or the launch?"""
import statistics, sys
import torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG


def ns(a, R=10000):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(20_000_000)
    e0.record(); RG.run_regions(a, 1, 32, R); e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) * 1e6 / R


keep = []
fresh = []
for i in range(12):
    a = torch.zeros(32 + 4096 * i, dtype=torch.float64, device="cuda")  # a different address each time
    keep.append(a)
    RG.run_regions(a, 1, 32, 10)
    fresh.append((hex(a.data_ptr()), round(ns(a), 1)))
same = [round(ns(keep[0]), 1) for _ in range(12)]
print("fresh allocations:", fresh)
print("same array, 12 launches:", same)
