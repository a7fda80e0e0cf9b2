"""Model files and signal files for the render path.

* ``load_model`` / ``save_model`` read and write the reference's single-file
  JSON model (``seminmf.py:300-380``, format version 1): ``f`` is the
  resonance filter, ``G`` either a dense row-major ``[N][K]`` list or, for a
  sparsified model, one ``{"indices", "values"}`` object per direction.
  Errors and messages follow the reference (``DataError``).
* ``load_renderer`` turns one JSON model per ear straight into the
  device-resident tap tables of :class:`batch.BatchRenderer` (one upload of
  the ELL table, f per ear), the object every batched GPU entry point uses.
* ``read_signal`` / ``write_signal`` are the reference's mono signal I/O
  (``hrir_io.py:274-357``): PCM16 or float32 WAV by extension, otherwise
  headerless little-endian float32 with an explicit rate.
"""
from __future__ import annotations

import json
import struct

import numpy as np

from .errors import DataError
from .types import FactorizedModel, Signal, SparseFilter

MODEL_FORMAT_VERSION = 1  # seminmf.py:38
_SPARSIFY_KEYS = ("lambda", "transform", "prune_threshold", "per_direction")


# ------------------------------------------------------------------ models ----
def load_model(path: str) -> FactorizedModel:
    """Read a model written by :func:`save_model` (ref: seminmf.py:336-380)."""
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except FileNotFoundError:
        raise DataError("no model file at %s" % path) from None
    except json.JSONDecodeError as exc:
        raise DataError("model file is not valid JSON: %s" % exc) from None
    if not isinstance(doc, dict) or doc.get("format_version") != MODEL_FORMAT_VERSION or "f" not in doc:
        raise DataError("%s is not a recognized model file" % path)
    G = doc["G"]
    info = None
    if G and isinstance(G[0], dict):
        K = int(doc["K"])
        reflections = [SparseFilter(indices=np.asarray(e["indices"], dtype=np.int64),
                                    values=np.asarray(e["values"], dtype=np.float64), length=K) for e in G]
        info = {k: doc[k] for k in _SPARSIFY_KEYS if k in doc} or None
    else:
        reflections = np.asarray(G, dtype=np.float64)
    model = FactorizedModel(
        resonance_taps=np.asarray(doc["f"], dtype=np.float64),
        reflections=reflections,
        sample_rate_hz=float(doc.get("sample_rate_hz", 0.0)),
        directions=list(doc.get("directions", [])),
        seed=int(doc.get("seed", 0)),
        rmse_history=list(doc.get("training_log", [])),
        sparsify_info=info,
    )
    if model.num_taps != doc["M"] or model.num_directions != doc["N"]:
        raise DataError("model dimensions disagree with the stored metadata")
    return model


def save_model(model: FactorizedModel, path: str) -> None:
    """Write ``model`` in the reference's JSON layout (ref: seminmf.py:300-333)."""
    if model.is_sparse:
        G = [{"indices": [int(i) for i in r.indices], "values": [float(v) for v in r.values]}
             for r in model.reflections]
    else:
        G = np.asarray(model.reflections, dtype=np.float64).tolist()
    doc = {
        "format_version": MODEL_FORMAT_VERSION,
        "M": model.num_taps,
        "N": model.num_directions,
        "K": model.reflection_length,
        "sample_rate_hz": float(model.sample_rate_hz),
        "seed": int(model.seed),
        "f": np.asarray(model.resonance_taps, dtype=np.float64).tolist(),
        "G": G,
        "training_log": [float(v) for v in model.rmse_history],
        "directions": list(model.directions),
    }
    if model.sparsify_info:
        doc.update(model.sparsify_info)
    with open(path, "w") as fh:
        json.dump(doc, fh)
        fh.write("\n")


def load_renderer(paths):
    """One JSON model per ear -> :class:`batch.BatchRenderer` (device tap tables).

    All ears must share direction count, reflection length and resonance
    length (the fused kernel renders every (ear, direction) row at once).
    """
    from .batch import BatchRenderer

    if isinstance(paths, str):
        paths = [paths]
    return BatchRenderer([load_model(p) for p in paths])


# ----------------------------------------------------------------- signals ----
def read_signal(path: str, sample_rate_hz: float | None = None) -> Signal:
    """Mono WAV (by extension) or headerless float32 (ref: hrir_io.py:274-288)."""
    if path.lower().endswith(".wav"):
        return _read_wav(path)
    if sample_rate_hz is None:
        raise DataError("headerless signal files need an explicit sample rate")
    try:
        raw = np.fromfile(path, dtype="<f4")
    except FileNotFoundError:
        raise DataError("no such file: %s" % path) from None
    return Signal(samples=raw.astype(np.float64), sample_rate_hz=sample_rate_hz)


def write_signal(signal: Signal, path: str) -> None:
    """Mono float32 WAV (by extension) or headerless float32 (ref: hrir_io.py:291-296)."""
    if path.lower().endswith(".wav"):
        _write_wav_float32(np.asarray(signal.samples), float(signal.sample_rate_hz), path)
    else:
        np.asarray(signal.samples, dtype="<f4").tofile(path)


def _read_wav(path: str) -> Signal:
    """RIFF walk: fmt + data chunks, word-aligned (ref: hrir_io.py:299-334)."""
    try:
        with open(path, "rb") as fh:
            blob = fh.read()
    except FileNotFoundError:
        raise DataError("no such file: %s" % path) from None
    if len(blob) < 12 or blob[0:4] != b"RIFF" or blob[8:12] != b"WAVE":
        raise DataError("%s is not a RIFF/WAVE file" % path)
    chunks = {}
    at = 12
    while at + 8 <= len(blob):
        tag = blob[at:at + 4]
        (n,) = struct.unpack_from("<I", blob, at + 4)
        chunks[tag] = blob[at + 8:at + 8 + n]  # a repeated chunk overrides, as in the reference
        at += 8 + n + (n & 1)
    if b"fmt " not in chunks or b"data" not in chunks:
        raise DataError("%s is missing its fmt or data chunk" % path)
    fmt_code, channels, rate, _, _, bits = struct.unpack_from("<HHIIHH", chunks[b"fmt "])
    if channels != 1:
        raise DataError("only mono WAV is supported, got %d channels" % channels)
    data = chunks[b"data"]
    if fmt_code == 1 and bits == 16:
        samples = np.frombuffer(data, dtype="<i2").astype(np.float64) / 32768.0
    elif fmt_code == 3 and bits == 32:
        samples = np.frombuffer(data, dtype="<f4").astype(np.float64)
    else:
        raise DataError("unsupported WAV encoding (format %d, %d bits); use PCM16 or float32" % (fmt_code, bits))
    return Signal(samples=samples, sample_rate_hz=float(rate))


def _write_wav_float32(samples: np.ndarray, rate_hz: float, path: str) -> None:
    """IEEE-float mono WAV with a fact chunk (ref: hrir_io.py:337-357)."""
    body = np.asarray(samples, dtype="<f4").tobytes()
    rate = int(round(rate_hz))
    fmt = struct.pack("<HHIIHH", 3, 1, rate, 4 * rate, 4, 32)
    parts = [b"WAVE",
             b"fmt " + struct.pack("<I", len(fmt)) + fmt,
             b"fact" + struct.pack("<II", 4, samples.size),
             b"data" + struct.pack("<I", len(body)) + body]
    payload = b"".join(parts)
    with open(path, "wb") as fh:
        fh.write(b"RIFF" + struct.pack("<I", len(payload)) + payload)
