"""Per-call latency of the reference-shaped API (engine.render / Renderer.render) on cfg1 shapes."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_03162_b200 import engine, synth
cfg = synth.CONFIGS["cfg2"]  # 1,250 directions; cfg1 signal length below
ms = synth.models(cfg, seed=1)
y = synth.source(44_100, seed=2)
r = engine.Renderer(ms[0])
for i in range(5): r.render(y, i)
torch.cuda.synchronize()
yt = torch.from_numpy(y.astype(np.float32)).cuda()
for label, fn, ndir in [("engine.render (new Renderer each call)", lambda d: engine.render(ms[0], y, d), 4),
                        ("Renderer.render, first call per direction", lambda d: r.render(y, d), 1250),
                        ("Renderer.render, repeated directions", lambda d: r.render(y, d), 4),
                        ("Renderer.render torch in/out, repeated", lambda d: r.render(yt, d), 4)]:
    if ndir != 1250:
        for i in range(5):  # warm: plans and the y*f cache for this input type
            fn(i % ndir)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 50
    for i in range(n):
        out = fn(100 + i if ndir == 1250 else i % ndir)
    torch.cuda.synchronize()
    print("%-45s %.3f ms/call" % (label, (time.perf_counter() - t0) / n * 1e3))

# ConvPlan / convolve in each mode (plan built once; numpy in/out)
taps = np.random.default_rng(3).standard_normal(200)
for mode, bs in [("dense_direct", None), ("fft_overlap_save", 1024), ("fft_overlap_save", 4096)]:
    plan = engine.ConvPlan(taps, mode, block_size=bs)
    for i in range(5):
        engine.convolve(plan, y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(50):
        engine.convolve(plan, y)
    print("%-45s %.3f ms/call" % ("convolve %s%s" % (mode, "" if bs is None else " block %d" % bs),
                                  (time.perf_counter() - t0) / 50 * 1e3))
sp = engine.ConvPlan(ms[0].reflections[0], "sparse_direct")
for i in range(5):
    engine.convolve(sp, y)
t0 = time.perf_counter()
for i in range(50):
    engine.convolve(sp, y)
print("%-45s %.3f ms/call" % ("convolve sparse_direct (K=100, nnz 16)", (time.perf_counter() - t0) / 50 * 1e3))
