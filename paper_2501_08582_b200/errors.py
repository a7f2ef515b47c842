"""Exception vocabulary of the reference (/root/reference/pkg/src/lors/errors.py:4-30).

The C-ABI status codes map onto these: LORS_ERR_SHAPE -> ShapeError,
LORS_ERR_ARGUMENT -> ArgumentError, device/CUDA failures -> DeviceError
(a RuntimeError).
"""


class ShapeError(ValueError):
    """Operand shapes are incompatible (errors.py:4-5)."""


class ArgumentError(ValueError):
    """Invalid argument values: rank, alpha, variant, dropout (errors.py:8-9)."""


class NumericError(ArithmeticError):
    """Non-finite result (errors.py:12-23)."""

    def __init__(self, message, residual=None, step=None):
        super().__init__(message)
        self.residual = residual
        self.step = step


class GraphError(RuntimeError):
    """Backward context reused (errors.py:26-27; adapters.py:197-200)."""


class CheckpointFormatError(Exception):
    """Malformed checkpoint file (errors.py:29-30)."""


class DeviceError(RuntimeError):
    """Not an sm_100 device, the native library is missing, or a CUDA launch failed."""
