"""Per-block device latency of the streaming step only (cfg4 shapes), for A/B builds."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_03162_b200 import batch, synth  # noqa: E402

cfg = synth.CONFIGS["cfg4"]
ms = synth.models(cfg, seed=4)
sd = synth.source_directions(cfg.sources, cfg.dirs, seed=4)
y = synth.device_sources(cfg.sources, 256 * 400, seed=44)
st = batch.StreamRenderer(ms, sd, 256)
out = torch.empty((2, 256 * 400), device="cuda")
lat = []
for b in range(400):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200_000)
    e0.record()
    st.step(y[:, b * 256:(b + 1) * 256], out=out[:, b * 256:(b + 1) * 256])
    e1.record()
    e1.synchronize()
    lat.append(e0.elapsed_time(e1) * 1e3)
print("median %.2f us" % statistics.median(lat[20:]))
