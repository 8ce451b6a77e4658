"""Region programs with device-malloc args lists, one launch per line, for
compute-sanitizer triage (measurement tool, not product)."""
import sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import golden_util as G
from paper_1711_10413_b200 import program as PG
from test_program import our_layouts, launches
stem, t, w = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
if len(sys.argv) > 4:  # per-thread stack limit in bytes (cudaLimitStackSize)
    import ctypes
    torch.zeros(1, device="cuda")
    rt = ctypes.CDLL("libcudart.so.12")
    print("set stack limit", int(sys.argv[4]), rt.cudaDeviceSetLimit(0, ctypes.c_size_t(int(sys.argv[4]))))
p = next(x for x in G.load("corpus") if x["stem"] == stem)
prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda") for _, sz, init in prog.buffers]
out = PG.run_program(prog, bufs, prealloc_entries=20, list_allocator=1)
torch.cuda.synchronize()
st = out.team_stats()
print(stem, t, w, [(s.trap, s.dynamic_allocs, s.dynamic_frees) for s in st][:2], [len(r.captures) for r in prog.regions])
