"""B200-native LARS data-parallel step (arXiv 1709.05011 hot path).

Drop-in for the reference `batchlab.optim` step API over device-resident,
flat, layer-segmented fp32 buffers; the step is one hand-written sm_100a
kernel (`csrc/lars_kernels.cu`) behind the C ABI of `include/lars_b200.h`,
and the sharded multi-GPU step adds NCCL reduce-scatter / all-gather
(`cluster.py`).
"""

from . import errors, layouts
from .errors import (BatchLabError, ConfigError, ConsistencyError, DivergenceError, NativeError,
                     ProtocolError, ScheduleExhaustedError)

__all__ = [
    "errors", "layouts", "BatchLabError", "ConfigError", "ConsistencyError", "DivergenceError",
    "NativeError", "ProtocolError", "ScheduleExhaustedError",
]
