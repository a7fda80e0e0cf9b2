"""One tensor-core mixdown partial at cfg5 laws for ncu (T reduced to keep replays cheap).

    ncu --set full --import-source on -k regex:k_mix_mma --launch-skip 2 --launch-count 1 \
        -o gpurun_out/mix python tools/ncu_mix.py [T]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1502_03162_b200 import batch, synth  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 720_000
cfg = synth.CONFIGS["cfg5"]
ms = synth.models(cfg, seed=5)
sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
y = synth.device_sources(cfg.sources, T, seed=1000)
mix = batch.MixRenderer(ms, sd, T)
z = mix.alloc_z()
for _ in range(2):
    mix.partial(y, z=z, check_finite=False)
torch.cuda.synchronize()
print("path", mix.path)
