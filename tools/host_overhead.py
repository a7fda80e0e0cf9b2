"""Host-side cost of one BatchRenderer.render_all call (enqueue only) vs its device time."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_03162_b200 import batch, synth  # noqa: E402

cfg = synth.CONFIGS["cfg2"]
ms = synth.models(cfg, seed=2)
br = batch.BatchRenderer(ms)
y = torch.from_numpy(synth.source(55_000, seed=1).astype(np.float32)).cuda()
out = br.alloc(y.numel())
for _ in range(5):
    br.render_all(y, out=out, check_finite=False)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    br.render_all(y, out=out, check_finite=False)
t_enq = (time.perf_counter() - t0) / n
torch.cuda.synchronize()
t_all = (time.perf_counter() - t0) / n
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(2_000_000)
e0.record()
for _ in range(n):
    br.render_all(y, out=out, check_finite=False)
e1.record()
torch.cuda.synchronize()
print("host enqueue %.1f us/call, wall %.1f us/call, device (queued back-to-back) %.1f us/call"
      % (t_enq * 1e6, t_all * 1e6, e0.elapsed_time(e1) / n * 1e3))
