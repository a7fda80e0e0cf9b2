"""Sustained power / SM clock while the cfg5 mixdown runs back to back (vs a plain HBM copy).

    python tools/power_probe.py
"""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_1502_03162_b200 import batch, synth  # noqa: E402


def sample(fn, seconds=4.0):
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    pw, clk, stop = [], [], threading.Event()

    def run():
        while not stop.is_set():
            pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.01)
    t = threading.Thread(target=run)
    t.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    n = 0
    t0 = time.time()
    ev[0].record()
    while time.time() - t0 < seconds:
        fn()
        n += 1
        if n % 8 == 0:
            torch.cuda.synchronize()
    ev[1].record()
    torch.cuda.synchronize()
    stop.set()
    t.join()
    ms = ev[0].elapsed_time(ev[1]) / n
    k = len(pw) // 3  # steady state: last two thirds
    return ms, statistics.median(pw[k:]), statistics.median(clk[k:])


if __name__ == "__main__":
    torch.cuda.set_device(0)
    cfg = synth.CONFIGS["cfg5"]
    ms = synth.models(cfg, seed=5)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
    y = synth.device_sources(cfg.sources, cfg.ny, seed=1000)
    dst = torch.empty(y.numel() // 4, device="cuda")
    src = y.view(-1)[: dst.numel()]
    print("copy 1/4 of y (23.6 GB moved): ms %.3f  W %.0f  MHz %.0f" % sample(lambda: dst.copy_(src)), flush=True)
    print("read-only sum of y (47 GB): ms %.3f  W %.0f  MHz %.0f" % sample(lambda: y.sum()), flush=True)
    for env in ("1", "0"):
        os.environ["TOEP_MIX_MMA"] = env
        mix = batch.MixRenderer(ms, sd, cfg.ny)
        z = mix.alloc_z()
        mix.partial(y, z=z, check_finite=False)
        print("mix %s: ms %.3f  W %.0f  MHz %.0f" % ((mix.path,) + sample(lambda: mix.partial(y, z=z, check_finite=False))),
              flush=True)
