"""A few cfg4 streaming steps, one at a time (for TOEP_STREAM_PROF builds: phase timestamps per block)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1502_03162_b200 import batch, synth  # noqa: E402

cfg = synth.CONFIGS["cfg4"]
ms = synth.models(cfg, seed=4)
sd = synth.source_directions(cfg.sources, cfg.dirs, seed=4)
B = cfg.block
y = synth.device_sources(cfg.sources, 40 * B, seed=44)
st = batch.StreamRenderer(ms, sd, B)
out = torch.empty((cfg.ears, 40 * B), device="cuda")
for b in range(40):
    st.step(y[:, b * B:(b + 1) * B], out=out[:, b * B:(b + 1) * B])
    torch.cuda.synchronize()
