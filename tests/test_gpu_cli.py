"""GPU: model JSON -> device tap tables and the CLI render / render-all / bench
subcommands, against the reference's own renders of the golden model files
(tests/golden/make_io_golden.py) at the north_star tolerance."""
import json
import os

import numpy as np
import pytest

from conftest import TOL, rel_l2
from paper_1502_03162_b200 import model_io
from paper_1502_03162_b200.cli import main

pytestmark = pytest.mark.gpu
IO = os.path.join(os.path.dirname(__file__), "golden", "io")
GOLD = np.load(os.path.join(IO, "io_golden.npz"))


@pytest.mark.parametrize("name", ["model_sparse", "model_dense"])
def test_load_renderer_matches_reference_render(cuda, name):
    br = model_io.load_renderer(os.path.join(IO, name + ".json"))
    out = br.render_all(GOLD["y"]).cpu().numpy()[0]
    ref = GOLD[name + "_render"]
    assert out.shape == ref.shape
    for d in range(ref.shape[0]):
        assert rel_l2(out[d], ref[d]) <= TOL


@pytest.mark.parametrize("mode", ["sparse_direct", "dense_direct", "fft_overlap_save"])
def test_cli_render_matches_reference(cuda, tmp_path, mode):
    out = tmp_path / "o.wav"
    # sig_f32.wav holds GOLD["y"] rounded to float32, which the reference renders read back as well
    assert main(["render", os.path.join(IO, "model_sparse.json"), os.path.join(IO, "sig_f32.wav"),
                 "--direction", "2", "--out", str(out), "--mode", mode]) == 0
    got = model_io.read_signal(str(out)).samples
    m = model_io.load_model(os.path.join(IO, "model_sparse.json"))
    y32 = GOLD["sig_f32"]
    expected = np.convolve(y32, np.convolve(m.resonance_taps, m.reflection(2)))
    assert got.size == expected.size
    assert rel_l2(got, expected) <= TOL
    run = json.load(open(tmp_path / "run.json"))
    assert run["subcommand"] == "render" and run["config"]["mode"] == mode


def test_cli_render_all_two_ears(cuda, tmp_path):
    out = tmp_path / "all.npy"
    models = [os.path.join(IO, "model_sparse.json"), os.path.join(IO, "model_dense.json")]
    with pytest.raises(SystemExit):  # headerless input without a rate is a usage error
        main(["render-all", *models, "--signal", str(tmp_path / "x.f32"), "--out", str(out)])
    assert main(["render-all", *models, "--signal", os.path.join(IO, "sig_pcm16.wav"), "--out", str(out)]) == 0
    got = np.load(out)
    y = GOLD["sig_pcm16"]
    assert got.shape[:2] == (2, 5)
    for e, path in enumerate(models):
        m = model_io.load_model(path)
        for d in range(5):
            ref = np.convolve(y, np.convolve(m.resonance_taps, m.reflection(d)))
            assert rel_l2(got[e, d], ref) <= TOL


def test_cli_bench_csv(cuda, tmp_path):
    out = tmp_path / "bench.csv"
    assert main(["bench", "--signal-len", "256", "--nnze", "2,8", "--repeats", "3", "--out", str(out)]) == 0
    lines = open(out).read().splitlines()
    assert lines[0] == "mode,signal_len,nnze,block_size,ns_per_sample_median,flops_model"
    assert len(lines) == 1 + 2 * 3
    run = json.load(open(tmp_path / "run.json"))
    assert run["latency"]["default_backend"] == "cuda"
    assert main(["bench", "--signal-len", "128", "--nnze", "4", "--repeats", "3", "--compare-backends",
                 "--out", str(out)]) == 0
    assert open(out).read().splitlines()[0].endswith(",backend")
