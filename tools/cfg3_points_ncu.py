"""Per-point ncu evidence for the config-3 sweep (17 points, 1,250 directions x 2 ears).

On the GPU box:
    ncu --profile-from-start off --clock-control none --csv \
        --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --log-file gpurun_out/r2/cfg3_points.csv \
        python tools/cfg3_points_ncu.py run > gpurun_out/r2/cfg3_points.jsonl
Here:
    python tools/cfg3_points_ncu.py summarize gpurun_out/r2/cfg3_points.csv gpurun_out/r2/cfg3_points.jsonl

`run` renders every point twice unprofiled, then once between
cudaProfilerStart/Stop, and prints one JSON line per point with the number of
launches that render made (br.native.kernels), so `summarize` can cut the
serialised launch list into points.  ncu times are cold-cache and serialised
(the fill launch no longer overlaps the main one): they show each point's
DRAM traffic against its algorithmic bytes, not its bench time.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run():
    import numpy as np
    import torch

    from paper_1502_03162_b200 import batch, synth

    cudart = torch.cuda.cudart()
    for cfg in synth.cfg3_points():
        ms = synth.models(cfg, seed=cfg.K * 1000 + cfg.nnz)
        y = torch.from_numpy(synth.source(cfg.ny, seed=3).astype(np.float32)).cuda()
        br = batch.BatchRenderer(ms)
        out = br.alloc(cfg.ny)
        for _ in range(2):
            br.render_all(y, out=out, check_finite=False)
        torch.cuda.synchronize()
        cudart.cudaProfilerStart()
        br.render_all(y, out=out, check_finite=False)
        torch.cuda.synchronize()
        cudart.cudaProfilerStop()
        L = br.out_len(cfg.ny)
        print(json.dumps({"point": cfg.name, "K": cfg.K, "nnz": cfg.nnz, "path": br.native.path(),
                          "launches": br.native.kernels(cfg.ny), "alg_bytes": 4.0 * cfg.ears * cfg.dirs * L + 4 * cfg.ny}),
              flush=True)
        del out, br


def _launches(path):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    # one dict per launch: {metric: value}
    by = {}
    order = []
    for r in rows:
        key = r["ID"]
        if key not in by:
            by[key] = {"name": r["Kernel Name"]}
            order.append(key)
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        by[key][r["Metric Name"]] = v * scale
    return [by[k] for k in order]


def summarize(csv_path, jsonl_path):
    pts = [json.loads(ln) for ln in open(jsonl_path) if ln.strip().startswith("{")]
    ls = _launches(csv_path)
    print("cfg3 per-point ncu (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum; "
          "one render per point, launches serialised): %s" % csv_path)
    print("%-18s %-7s %4s %9s %9s %9s %9s %8s  kernels" % ("point", "path", "n", "sum_us", "max_us", "alg_MB",
                                                           "dram_MB", "dram/alg"))
    i = 0
    for p in pts:
        mine = ls[i:i + p["launches"]]
        i += p["launches"]
        t = sum(k.get("gpu__time_duration.sum", 0.0) for k in mine)
        dram = sum(k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0) for k in mine)
        names = ",".join(sorted({k["name"].split("(")[0].replace("void ", "").replace("toep::", "")
                                 for k in mine}))
        # the fill launch overlaps the main one outside ncu: the longest launch is the critical path
        tmax = max((k.get("gpu__time_duration.sum", 0.0) for k in mine), default=0.0)
        print("%-18s %-7s %4d %9.1f %9.1f %9.1f %9.1f %8.3f  %s" % (
            p["point"], p["path"], len(mine), t / 1e3, tmax / 1e3, p["alg_bytes"] / 1e6, dram / 1e6,
            dram / p["alg_bytes"], names))
    if i != len(ls):
        print("warning: %d launches in the csv, %d attributed" % (len(ls), i))


if __name__ == "__main__":
    if sys.argv[1:2] == ["run"]:
        run()
    elif sys.argv[1:2] == ["summarize"]:
        summarize(sys.argv[2], sys.argv[3])
    else:
        raise SystemExit(__doc__)
