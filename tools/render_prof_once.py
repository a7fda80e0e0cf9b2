"""Three renders of one config-2/3 point (for TOEP_MMA_PROF builds: per-role wait counters).

    python tools/render_prof_once.py [K nnz]     # default: cfg2 (K=100, nnz=16)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_03162_b200 import batch, synth  # noqa: E402
from paper_1502_03162_b200.synth import Config  # noqa: E402

K, nnz = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (100, 16)
cfg = Config("p", ny=441_000, M=200, K=K, nnz=nnz, dirs=1250, ears=2)
ms = synth.models(cfg, seed=K * 1000 + nnz)
br = batch.BatchRenderer(ms)
y = torch.from_numpy(synth.source(cfg.ny, seed=3).astype(np.float32)).cuda()
out = br.alloc(cfg.ny)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(3):
    ev[0].record()
    br.render_all(y, out=out, check_finite=False)
    ev[1].record()
    torch.cuda.synchronize()
print("K %d nnz %d path %s: %.3f ms" % (K, nnz, br.native.path(), ev[0].elapsed_time(ev[1])))
