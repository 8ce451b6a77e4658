"""Config-3 kernel on one team (96 workers, 2000 nested regions) with the
frames in the warps' shared-memory slots (argv[1] = slot bytes, default
2048) or, with 0, on the global overflow chain -- for ncu (measurement
tool, not product)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG  # noqa: E402

slot = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
a = torch.zeros(96, dtype=torch.float64, device="cuda")
RG.run_nested(a, 1, 96, 10, warp_slot_bytes=slot, collect=False)
RG.run_nested(a, 1, 96, 2000, warp_slot_bytes=slot, collect=False)
torch.cuda.synchronize()
print("nested overflow probe done", slot)
