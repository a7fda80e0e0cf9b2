"""B200-native sparse-HRIR renderer (arXiv 1502.03162 render path).

Drop-in for the render path of the reference ``toepnmf`` package: the
``engine`` module mirrors ``toepnmf.engine``; ``batch`` adds the fused
all-directions renderer, the reflection-first mixdown and the streaming
block mode; ``dist`` shards the mixdown over GPUs with one NCCL reduce.
All arithmetic runs in the sm_100a kernels of ``libtoep_b200.so``.
"""
from . import engine
from .errors import DataError, NumericalError, ToepnmfError
from .types import FactorizedModel, Signal, SparseFilter

__all__ = ["engine", "DataError", "NumericalError", "ToepnmfError", "FactorizedModel", "Signal", "SparseFilter"]
__version__ = "0.1.0"
