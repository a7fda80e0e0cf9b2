"""Generate golden vectors from the *reference itself* (run in the dev container).

    python tests/golden/make_golden.py

Imports the read-only reference package from /root/reference/pkg/src, with its
compiled Cython kernels supplied by oracle/_ref (built from
pkg/src/toepnmf/engine/_kernels.pyx by oracle/Makefile), and records what the
reference's public API returns on small seeded inputs.  The fixtures are the
parity anchor on the GPU box, where /root/reference does not exist.

Every array is produced by reference code paths:
  * engine.convolve / ConvPlan for the known-answer tests of
    pkg/tests/test_engine.py:44-56,82-85,128-146
  * engine.Renderer(...).render + counters (engine/__init__.py:208-269)
  * numpy fp64 sums of Renderer.render for the mixdown composition
  * the cost model (engine/__init__.py:278-313)
"""
import glob
import importlib.machinery
import importlib.util
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"


def load_reference():
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, ROOT)
    cands = glob.glob(os.path.join(ROOT, "oracle", "_ref", "_kernels*.so"))
    if cands:  # make the reference's compiled backend importable as toepnmf.engine._kernels
        loader = importlib.machinery.ExtensionFileLoader("toepnmf.engine._kernels", cands[0])
        spec = importlib.util.spec_from_file_location("toepnmf.engine._kernels", cands[0], loader=loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        sys.modules["toepnmf.engine._kernels"] = mod
    import toepnmf.engine as engine
    import toepnmf.seminmf as seminmf
    import toepnmf.sparsify as sparsify
    return engine, seminmf, sparsify


def main():
    engine, seminmf, sparsify = load_reference()
    from paper_1502_03162_b200 import synth

    out = {}
    backends = engine.available_backends()
    out["backends"] = np.array(backends)
    out["default_backend"] = np.array(engine.DEFAULT_BACKEND)

    # --- known-answer tests (pkg/tests/test_engine.py:44-56)
    kat = {
        "identity": (np.array([1.0]), np.array([3.0, -1.0, 2.0])),
        "pinned_small": (np.array([1.0, 2.0]), np.array([3.0, 4.0])),
    }
    for name, (taps, y) in kat.items():
        for mode in engine.MODES:
            plan = engine.ConvPlan(taps, mode, backend="compiled")
            out["kat_%s_%s" % (name, mode)] = engine.convolve(plan, y)
            out["kat_%s_%s_macs" % (name, mode)] = np.array(plan.macs)
    sf = sparsify.SparseFilter(np.array([0, 3]), np.array([1.0, 2.0]), 4)
    plan = engine.ConvPlan(sf, "sparse_direct", backend="compiled")
    out["kat_pinned_sparse"] = engine.convolve(plan, np.array([1.0, 1.0, 1.0]))
    out["kat_pinned_sparse_macs"] = np.array(plan.macs)

    # --- random conv cases incl. degenerate lengths, both kernels
    rng = np.random.default_rng(20261019)
    cases = [(1, 1), (1, 17), (17, 1), (5, 11), (101, 441), (300, 50)]
    for i, (nt, ny) in enumerate(cases):
        taps = rng.standard_normal(nt).astype(np.float32).astype(np.float64)
        y = rng.standard_normal(ny).astype(np.float32).astype(np.float64)
        out["dense_%d_taps" % i] = taps
        out["dense_%d_y" % i] = y
        out["dense_%d_out" % i] = engine.convolve(engine.ConvPlan(taps, "dense_direct", backend="compiled"), y)
    for i, (length, nnz, ny) in enumerate([(1, 1, 10), (4, 2, 3), (100, 16, 500), (150, 64, 300), (600, 40, 700),
                                            (12, 0, 9)]):
        idx = np.sort(rng.choice(length, nnz, replace=False)).astype(np.int64)
        vals = np.abs(rng.standard_normal(nnz)).astype(np.float32).astype(np.float64) + 0.01
        vals = vals.astype(np.float32).astype(np.float64)
        y = rng.standard_normal(ny).astype(np.float32).astype(np.float64)
        sfi = sparsify.SparseFilter(idx, vals, length)
        plan = engine.ConvPlan(sfi, "sparse_direct", backend="compiled")
        out["sparse_%d_idx" % i] = idx
        out["sparse_%d_vals" % i] = vals
        out["sparse_%d_len" % i] = np.array(length)
        out["sparse_%d_y" % i] = y
        out["sparse_%d_out" % i] = engine.convolve(plan, y)
        out["sparse_%d_macs" % i] = np.array(plan.macs)

    # --- BASELINE config 1, full size, through the reference Renderer
    cfg = synth.CONFIGS["cfg1"]
    ms = synth.models(cfg, seed=1)
    y = synth.source(cfg.ny, seed=11)
    ref_model = seminmf.FactorizedModel(ms[0].resonance_taps,
                                        [sparsify.SparseFilter(r.indices, r.values, r.length) for r in ms[0].reflections])
    r = engine.Renderer(ref_model, backend="compiled")
    out["cfg1_y_sum"] = np.array([y.sum(), np.abs(y).sum(), y[:1000].std()])  # y regenerated from synth seed 11
    out["cfg1_f"] = ms[0].resonance_taps
    out["cfg1_idx"] = ms[0].reflections[0].indices
    out["cfg1_vals"] = ms[0].reflections[0].values
    out["cfg1_out"] = r.render(y, 0)
    c = r.counters
    out["cfg1_counters"] = np.array([c["resonance_macs"], c["reflection_macs"], c["cache_hits"], c["cache_misses"]])

    # --- multi-direction, two ears, sparse models (BASELINE laws, reduced size)
    cfg = synth.Config("g2", ny=1500, M=200, K=100, nnz=16, dirs=4, ears=2)
    ms = synth.models(cfg, seed=2)
    y = synth.source(cfg.ny, seed=22)
    rows = []
    for e, m in enumerate(ms):
        rm = seminmf.FactorizedModel(m.resonance_taps,
                                     [sparsify.SparseFilter(f.indices, f.values, f.length) for f in m.reflections])
        rr = engine.Renderer(rm, backend="compiled")
        for d in range(cfg.dirs):
            rows.append(rr.render(y, d))
        out["g2_f_%d" % e] = m.resonance_taps
        for d in range(cfg.dirs):
            out["g2_idx_%d_%d" % (e, d)] = m.reflections[d].indices
            out["g2_vals_%d_%d" % (e, d)] = m.reflections[d].values
        c = rr.counters
        out["g2_counters_%d" % e] = np.array([c["resonance_macs"], c["reflection_macs"], c["cache_hits"],
                                              c["cache_misses"]])
    out["g2_y"] = y.astype(np.float32)
    out["g2_out"] = np.stack(rows)

    # --- dense-reflection model (exact_model_data law, pkg/tests/conftest.py:31-42)
    rng2 = np.random.default_rng(10)
    f0 = rng2.standard_normal(24 - 6 + 1)
    f0[0] += 3.0
    G0 = rng2.uniform(0.1, 1.0, size=(4, 6))
    dm = seminmf.FactorizedModel(f0, G0)
    yd = np.random.default_rng(11).standard_normal(200)
    rd = engine.Renderer(dm, backend="compiled")
    out["dense_model_f"] = f0
    out["dense_model_G"] = G0
    out["dense_model_y"] = yd
    out["dense_model_out"] = np.stack([rd.render(yd, j) for j in range(4)])

    # --- mixdown composition: 12 sources x 2 ears, sum of reference renders (fp64)
    cfg = synth.Config("mx", ny=1200, M=200, K=100, nnz=24, dirs=9, ears=2, sources=10)
    ms = synth.models(cfg, seed=3)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=3)
    ys = np.stack([synth.source(cfg.ny, seed=100 + s) for s in range(cfg.sources)])
    mix = np.zeros((2, cfg.ny + cfg.M - 1))
    for e, m in enumerate(ms):
        rm = seminmf.FactorizedModel(m.resonance_taps,
                                     [sparsify.SparseFilter(f.indices, f.values, f.length) for f in m.reflections])
        rr = engine.Renderer(rm, backend="compiled")
        for s in range(cfg.sources):
            mix[e] += rr.render(ys[s], int(sd[s]))
        out["mx_f_%d" % e] = m.resonance_taps
        for d in range(cfg.dirs):
            out["mx_idx_%d_%d" % (e, d)] = m.reflections[d].indices
            out["mx_vals_%d_%d" % (e, d)] = m.reflections[d].values
    out["mx_y"] = ys.astype(np.float32)
    out["mx_dir"] = sd
    out["mx_out"] = mix

    # --- cost model (engine/__init__.py:278-313; pkg/tests/test_engine.py:284-325)
    out["cost_crossover"] = np.array([engine.time_domain_crossover(44100), engine.time_domain_crossover(2205)])
    out["cost_fft_25_44100"] = np.array(engine.cost_per_sample_fft(25, 44100))
    out["cost_fft_1024_1024"] = np.array(engine.cost_per_sample_fft(1024, 1024))

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
