"""Exception types of the reference interface (same names and bases).

InvalidPrimitiveError  core.py:21-22        (ValueError)
ResourceLimitError     rasterizer.py:28-29  (RuntimeError)
TrainingDiverged       optimizer.py:16-17   (RuntimeError)
"""


class InvalidPrimitiveError(ValueError):
    """Raised for Gaussian parameterizations that cannot form a valid primitive."""


class ResourceLimitError(RuntimeError):
    """Raised when a render would exceed the supported tile or instance count."""


class TrainingDiverged(RuntimeError):
    """Raised when the loss turns non-finite."""
