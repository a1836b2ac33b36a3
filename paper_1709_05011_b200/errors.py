"""Exception taxonomy of the LARS data-parallel step.

Mirrors the reference's error types (`pkg/src/batchlab/errors.py:4-49`) that the
optimizer step and the gradient aggregation raise, with the same constructor
signatures and attributes, so callers written against the reference catch the
same things.  `NativeError` is new: it wraps a non-zero status from the CUDA
C-ABI library (there is no native layer in the reference).
"""


class BatchLabError(Exception):
    """Base class for all package errors (`errors.py:4-5`)."""


class ConfigError(BatchLabError):
    """Invalid configuration / hyperparameters (`errors.py:8-9`)."""


class ConsistencyError(BatchLabError):
    """Replicas diverged where they must be identical (`errors.py:32-33`)."""


class ProtocolError(BatchLabError):
    """Shape mismatch between gradient sets in a collective (`errors.py:36-37`)."""


class ScheduleExhaustedError(BatchLabError):
    """Learning-rate schedule queried past its final iteration (`errors.py:40-41`)."""


class DivergenceError(BatchLabError):
    """Parameters became non-finite during an update (`errors.py:44-49`)."""

    def __init__(self, iteration, message=None):
        self.iteration = iteration
        super().__init__(message or f"non-finite update at iteration {iteration}")


class NativeError(BatchLabError):
    """The CUDA library returned a non-zero status code."""

    def __init__(self, code, message):
        self.code = code
        super().__init__(f"lars_b200 error {code}: {message}")
