"""Golden model/signal files written and read by the *reference itself*.

    python tests/golden/make_io_golden.py

Uses the read-only reference (``seminmf.save_model`` / ``load_model``,
``hrir_io.write_signal`` / ``read_signal``; seminmf.py:300-380,
hrir_io.py:274-357) to write small files into ``tests/golden/io/`` and records
what the reference reads back from each, so ``model_io`` and the CLI are
pinned against the reference's file formats on machines without it.
"""
import os
import sys
import wave

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_reference  # noqa: E402

OUT = os.path.join(HERE, "io")


def main():
    engine, seminmf, sparsify = load_reference()
    import toepnmf.hrir_io as hrir_io

    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(1502)
    lf, K, D = 9, 12, 5
    f = rng.standard_normal(lf) * np.exp(-np.arange(lf) / 3.0)
    sparse = []
    for _ in range(D):
        idx = np.sort(rng.choice(K, size=4, replace=False)).astype(np.int64)
        sparse.append(sparsify.SparseFilter(indices=idx, values=np.abs(rng.standard_normal(4)) + 0.1, length=K))
    m_sparse = seminmf.FactorizedModel(resonance_taps=f, reflections=sparse, sample_rate_hz=48000.0,
                                       directions=[(float(10 * i), 0.0) for i in range(D)], seed=7,
                                       rmse_history=[0.5, 0.25],
                                       sparsify_info={"lambda": 1e-3, "transform": "identity",
                                                      "prune_threshold": 1e-6, "per_direction": [1, 2, 3, 4, 5]})
    seminmf.save_model(m_sparse, os.path.join(OUT, "model_sparse.json"))
    dense = np.abs(rng.standard_normal((D, K))) * (rng.random((D, K)) < 0.5)
    m_dense = seminmf.FactorizedModel(resonance_taps=f[::-1].copy(), reflections=dense, sample_rate_hz=44100.0)
    seminmf.save_model(m_dense, os.path.join(OUT, "model_dense.json"))

    y = rng.standard_normal(300) * 0.5
    hrir_io.write_signal(hrir_io.Signal(samples=y, sample_rate_hz=8000.0), os.path.join(OUT, "sig_f32.wav"))
    pcm = np.clip(np.round(y * 20000), -32768, 32767).astype("<i2")
    with wave.open(os.path.join(OUT, "sig_pcm16.wav"), "wb") as w:
        w.setnchannels(1)
        w.setsampwidth(2)
        w.setframerate(22050)
        w.writeframes(pcm.tobytes())

    arrays = {}
    for name in ("model_sparse", "model_dense"):
        m = seminmf.load_model(os.path.join(OUT, name + ".json"))
        arrays[name + "_f"] = m.resonance_taps
        arrays[name + "_G"] = np.stack([m.reflection(i) for i in range(m.num_directions)])
        arrays[name + "_meta"] = np.array([m.num_taps, m.num_directions, m.reflection_length, m.sample_rate_hz])
        # reference render of every direction through the reference engine (compiled backend)
        arrays[name + "_render"] = np.stack([engine.Renderer(m).render(y, d) for d in range(m.num_directions)])
    for name in ("sig_f32", "sig_pcm16"):
        s = hrir_io.read_signal(os.path.join(OUT, name + ".wav"))
        arrays[name] = s.samples
        arrays[name + "_rate"] = np.array(s.sample_rate_hz)
    arrays["y"] = y
    np.savez_compressed(os.path.join(OUT, "io_golden.npz"), **arrays)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
