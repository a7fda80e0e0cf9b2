"""Input types of the render path.

Mirrors of the reference containers the engine consumes:
  * SparseFilter    <- pkg/src/toepnmf/sparsify.py:67-97
  * FactorizedModel <- pkg/src/toepnmf/seminmf.py:50-129 (render-relevant fields)
  * Signal          <- pkg/src/toepnmf/hrir_io.py:257-271
The engine only reads their attributes, so the reference's own objects can be
passed in unchanged (duck typing).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DataError


@dataclass
class SparseFilter:
    """A pruned reflection filter stored as index/value pairs (sparsify.py:67-97)."""

    indices: np.ndarray
    values: np.ndarray
    length: int

    def __post_init__(self):
        self.indices = np.asarray(self.indices, dtype=np.int64)
        self.values = np.asarray(self.values, dtype=np.float64)
        if self.indices.shape != self.values.shape or self.indices.ndim != 1:
            raise DataError("indices and values must be matching 1-d arrays")
        if self.indices.size:
            if np.any(np.diff(self.indices) <= 0):
                raise DataError("indices must be strictly increasing")
            if self.indices[0] < 0 or self.indices[-1] >= self.length:
                raise DataError("indices must lie in [0, %d)" % self.length)
            if not np.all(np.isfinite(self.values)) or np.any(self.values <= 0.0):
                raise DataError("values must be finite and positive")
        if self.length < 1:
            raise DataError("filter length must be at least 1")

    @property
    def nnze(self) -> int:
        return int(self.indices.size)

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.length)
        out[self.indices] = self.values
        return out


def is_sparse_filter(obj) -> bool:
    return all(hasattr(obj, a) for a in ("indices", "values", "length")) and not isinstance(obj, np.ndarray)


@dataclass
class FactorizedModel:
    """Resonance filter f plus per-direction reflection filters (seminmf.py:50-129).

    ``reflections`` is a dense (num_directions, K) non-negative array or a list
    of :class:`SparseFilter`.  One model describes one ear.
    """

    resonance_taps: np.ndarray
    reflections: object
    sample_rate_hz: float = 0.0
    directions: list = field(default_factory=list)
    seed: int = 0
    rmse_history: list = field(default_factory=list)
    sparsify_info: dict | None = None

    def __post_init__(self):
        self.resonance_taps = np.asarray(self.resonance_taps, dtype=np.float64)
        if self.resonance_taps.ndim != 1 or self.resonance_taps.size == 0:
            raise DataError("resonance taps must be a non-empty 1-d array")
        if not self.is_sparse:
            self.reflections = np.asarray(self.reflections, dtype=np.float64)
            if self.reflections.ndim != 2:
                raise DataError("dense reflections must be a 2-d array")
            if np.any(self.reflections < 0.0):
                raise DataError("reflection filters must be non-negative")
        if self.directions and len(self.directions) != self.num_directions:
            raise DataError("have %d direction entries for %d reflection filters"
                            % (len(self.directions), self.num_directions))

    @property
    def is_sparse(self) -> bool:
        return isinstance(self.reflections, list)

    @property
    def reflection_length(self) -> int:
        if self.is_sparse:
            return self.reflections[0].length
        return self.reflections.shape[1]

    @property
    def num_directions(self) -> int:
        return len(self.reflections)

    @property
    def num_taps(self) -> int:
        return self.resonance_taps.size + self.reflection_length - 1

    def reflection(self, i: int) -> np.ndarray:
        if self.is_sparse:
            return self.reflections[i].to_dense()
        return np.asarray(self.reflections[i], dtype=np.float64)

    def nnze(self, i: int) -> int:
        if self.is_sparse:
            return len(self.reflections[i].indices)
        return int(np.count_nonzero(self.reflections[i]))

    def reconstruct(self, directions=None) -> np.ndarray:
        if directions is None:
            directions = range(self.num_directions)
        out = np.empty((self.num_taps, len(directions)))
        for col, i in enumerate(directions):
            out[:, col] = np.convolve(self.resonance_taps, self.reflection(i))
        return out


@dataclass
class Signal:
    """A single-channel signal with its sample rate (hrir_io.py:257-271)."""

    samples: np.ndarray
    sample_rate_hz: float

    def __post_init__(self):
        self.samples = np.asarray(self.samples, dtype=np.float64)
        if self.samples.ndim != 1:
            raise DataError("signals are single-channel 1-d arrays")
        if not np.all(np.isfinite(self.samples)):
            raise DataError("signal contains non-finite samples")
        if self.sample_rate_hz <= 0:
            raise DataError("sample rate must be positive")
