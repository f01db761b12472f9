"""Exception types of the executor path, same names and meaning as the
reference (``svpart/executor.py:25-42``; CLI exit codes at ``cli.py:20-23``)."""


class ExecutorError(Exception):
    pass


class TooLarge(ExecutorError):
    pass


class PlanInvalid(ExecutorError):
    pass


class NonUnitaryDrift(ExecutorError):
    pass


class DimensionMismatch(ExecutorError):
    pass


class NativeError(RuntimeError):
    """The CUDA library reported a failure (or is missing on a GPU box)."""
