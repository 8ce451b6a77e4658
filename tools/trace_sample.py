"""A config-1 launch (2 teams x 64 workers, 6 regions, event log on) exported
as a Chrome/Perfetto trace to gpurun_out/ (measurement tool, not product)."""
import os, sys, torch
sys.path.insert(0, ".")
from paper_1711_10413_b200 import regions as RG
from paper_1711_10413_b200 import trace as TR
a = torch.zeros(2 * 64, dtype=torch.float64, device="cuda")
RG.run_regions(a, 2, 64, 6, max_events=1024)  # warm
out = RG.run_regions(a, 2, 64, 6, max_events=1024)
os.makedirs("gpurun_out", exist_ok=True)
TR.write_chrome_trace("gpurun_out/trace_config1.json", out.team_events(times=True))
print("trace written")
