"""bench.py's multi-rank launch path on CPU: ``--gpus N`` with no launcher
re-executes itself under torch.distributed.run with N processes; the ranks
rendezvous (gloo here, NCCL on GPUs) and split the config-5 sources by
direction.  Plus the config dicts both arms print (identical keys/values)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_n_spawns_n_ranks():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and len(d["shares"]) == 2
    assert sorted(s["rank"] for s in d["shares"]) == [0, 1]
    assert sum(s["sources"] for s in d["shares"]) == 4096
    assert d["config"]["workload"] == "cfg5"


def test_both_arms_print_the_same_config():
    sys.path.insert(0, ROOT)
    import bench
    for wl in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        for world in (1, 8):
            a = bench.workload_config(wl, world)
            b = json.loads(json.dumps(bench.workload_config(wl, world)))
            assert a == b and a["workload"] == wl
