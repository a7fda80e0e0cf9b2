"""Model JSON and signal files pinned against files the
reference itself wrote and read (tests/golden/make_io_golden.py), and the CLI's
host-side behaviour (usage and data errors, exit codes) -- no GPU needed."""
import json
import os

import numpy as np
import pytest

from conftest import has_gpu
from paper_1502_03162_b200 import DataError, FactorizedModel, Signal, SparseFilter, model_io
from paper_1502_03162_b200 import _lib
from paper_1502_03162_b200.cli import main

IO = os.path.join(os.path.dirname(__file__), "golden", "io")
GOLD = np.load(os.path.join(IO, "io_golden.npz"))


@pytest.mark.parametrize("name", ["model_sparse", "model_dense"])
def test_load_model_matches_reference(name):
    m = model_io.load_model(os.path.join(IO, name + ".json"))
    np.testing.assert_array_equal(m.resonance_taps, GOLD[name + "_f"])
    np.testing.assert_array_equal(np.stack([m.reflection(i) for i in range(m.num_directions)]), GOLD[name + "_G"])
    assert [m.num_taps, m.num_directions, m.reflection_length, m.sample_rate_hz] == list(GOLD[name + "_meta"])
    assert m.is_sparse == (name == "model_sparse")


def test_sparse_metadata_round_trip(tmp_path):
    m = model_io.load_model(os.path.join(IO, "model_sparse.json"))
    assert m.sparsify_info == {"lambda": 1e-3, "transform": "identity", "prune_threshold": 1e-6,
                               "per_direction": [1, 2, 3, 4, 5]}
    assert m.seed == 7 and m.rmse_history == [0.5, 0.25] and len(m.directions) == 5
    p = tmp_path / "again.json"
    model_io.save_model(m, str(p))
    a = json.load(open(os.path.join(IO, "model_sparse.json")))
    b = json.load(open(p))
    a["directions"] = [list(d) for d in a["directions"]]
    b["directions"] = [list(d) for d in b["directions"]]
    assert a == b  # byte-level layout aside, the documents are identical


def test_dense_round_trip(tmp_path):
    m = model_io.load_model(os.path.join(IO, "model_dense.json"))
    p = tmp_path / "d.json"
    model_io.save_model(m, str(p))
    assert json.load(open(p)) == json.load(open(os.path.join(IO, "model_dense.json")))


def test_load_model_errors(tmp_path):
    with pytest.raises(DataError, match="no model file"):
        model_io.load_model(str(tmp_path / "missing.json"))
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    with pytest.raises(DataError, match="not valid JSON"):
        model_io.load_model(str(bad))
    doc = json.load(open(os.path.join(IO, "model_sparse.json")))
    for patch, msg in (({"format_version": 2}, "not a recognized model file"),
                       ({"M": 99}, "disagree"), ({"N": 3}, "disagree")):
        p = tmp_path / "x.json"
        p.write_text(json.dumps({**doc, **patch}))
        with pytest.raises(DataError, match=msg):
            model_io.load_model(str(p))
    doc["G"][0]["indices"] = [3, 1, 2, 5]  # unsorted: SparseFilter validation
    p = tmp_path / "y.json"
    p.write_text(json.dumps(doc))
    with pytest.raises(DataError):
        model_io.load_model(str(p))


@pytest.mark.parametrize("name", ["sig_f32", "sig_pcm16"])
def test_read_wav_matches_reference(name):
    s = model_io.read_signal(os.path.join(IO, name + ".wav"))
    np.testing.assert_array_equal(s.samples, GOLD[name])
    assert s.sample_rate_hz == float(GOLD[name + "_rate"])


def test_signal_write_read(tmp_path):
    y = GOLD["y"]
    w = tmp_path / "o.wav"
    model_io.write_signal(Signal(samples=y, sample_rate_hz=8000.0), str(w))
    assert w.read_bytes() == open(os.path.join(IO, "sig_f32.wav"), "rb").read()  # same bytes as the reference
    r = tmp_path / "o.f32"
    model_io.write_signal(Signal(samples=y, sample_rate_hz=8000.0), str(r))
    s = model_io.read_signal(str(r), sample_rate_hz=8000.0)
    np.testing.assert_array_equal(s.samples, y.astype(np.float32))
    with pytest.raises(DataError, match="explicit sample rate"):
        model_io.read_signal(str(r))
    with pytest.raises(DataError, match="no such file"):
        model_io.read_signal(str(tmp_path / "none.wav"))
    (tmp_path / "junk.wav").write_bytes(b"RIFX0000WAVE")
    with pytest.raises(DataError, match="RIFF/WAVE"):
        model_io.read_signal(str(tmp_path / "junk.wav"))


def test_cli_usage_and_data_errors(tmp_path, capsys):
    assert main([]) == 2
    raw = tmp_path / "s.f32"
    np.zeros(8, "<f4").tofile(raw)
    with pytest.raises(SystemExit) as err:
        main(["render", os.path.join(IO, "model_sparse.json"), str(raw), "--direction", "0",
              "--out", str(tmp_path / "o.f32")])
    assert err.value.code == 2
    assert main(["render", str(tmp_path / "nomodel.json"), os.path.join(IO, "sig_f32.wav"), "--direction", "0",
                 "--out", str(tmp_path / "o.wav")]) == 3
    assert "data error" in capsys.readouterr().err
    assert main(["bench", "--nnze", "1,x", "--out", str(tmp_path / "b.csv")]) == 3


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_cli_render_without_gpu_fails_loudly(tmp_path):
    with pytest.raises(_lib.NativeUnavailable):
        main(["render", os.path.join(IO, "model_sparse.json"), os.path.join(IO, "sig_f32.wav"), "--direction", "1",
              "--out", str(tmp_path / "o.wav")])
