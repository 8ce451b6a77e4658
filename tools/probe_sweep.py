#!/usr/bin/env python
"""ompds_probe_overheads over frame sizes and depth patterns (one JSON)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_10413_b200 import regions as RG  # noqa: E402

out = {}
for fb, md in ((40, 2), (40, 4), (8, 1), (64, 4), (128, 2), (4, 3)):
    out[f"{fb}B_d{md}"] = RG.probe_overheads(16384, frame_bytes=fb, max_depth=md)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "probe_sweep.json", "w"), indent=1)
for k, v in out.items():
    print(k, v["pairs_per_iteration"], v["push_pop_pair_slot_cycles"], v["push_pop_pair_chain_cycles"],
          v["push_pop_pair_bookkeeping_cycles"], v["chain_vs_slot_per_pair_cycles"],
          v["cycles_per_iteration"])
