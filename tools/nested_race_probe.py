import os, sys, torch, ctypes as C
sys.path.insert(0, '.')
from paper_1711_10413_b200 import regions as RG
from paper_1711_10413_b200 import _lib as L
orig_sync = torch.cuda.synchronize
def run(nosync, side):
    st = torch.cuda.Stream() if side else torch.cuda.current_stream()
    teams = 1184
    a = torch.zeros(teams * 96, dtype=torch.float64, device='cuda')
    if nosync:
        torch.cuda.synchronize = lambda *a, **k: None
    RG.run_nested(a, teams, 96, 10, stream=st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); _, stacks = RG.run_nested(a, teams, 96, 2000, stream=st); e1.record(st)
    torch.cuda.synchronize = orig_sync
    e1.synchronize()
    print(f"nosync={nosync} side={side}: {e0.elapsed_time(e1)*1e6/2000:8.1f} ns  depth={stacks[0][0].max_depth}")
for ns in (False, True):
    for sd in (False, True):
        run(ns, sd)
