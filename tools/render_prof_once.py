import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1502_03162_b200 import batch, synth
cfg = synth.CONFIGS["cfg2"]
ms = synth.models(cfg, seed=2)
br = batch.BatchRenderer(ms)
y = torch.from_numpy(synth.source(cfg.ny, seed=3).astype(np.float32)).cuda()
out = br.alloc(cfg.ny)
for i in range(3):
    br.render_all(y, out=out, check_finite=False)
torch.cuda.synchronize()
