"""Exception taxonomy of the candidate-evaluation path and the mapping from
the native library's status codes onto it.

Mirrors convevo/errors.py:4-42 (same class names, base classes and extra
attributes) so callers catching ``ShapeError`` / ``EvalFailure`` keep working.
"""

__all__ = ["ShapeError", "EvalFailure", "FormatError", "ConfigError",
           "ProtocolError", "NativeError", "status_to_exception",
           "CE_OK", "CE_EINVAL", "CE_ENONFINITE", "CE_ENOMEM", "CE_ECUDA"]

# status codes of include/menndl_sm100.h
CE_OK, CE_EINVAL, CE_ENONFINITE, CE_ENOMEM, CE_ECUDA = 0, 1, 2, 3, 4


class ShapeError(ValueError):
    """A layer cannot consume (or would collapse) its input shape.

    ``layer_index``: offending layer position when known (repair() deletes it);
    ``dimension``: which dimension failed ("rows", "cols", "channels", "units").
    """

    def __init__(self, message, layer_index=None, dimension=None):
        ValueError.__init__(self, message)
        self.layer_index, self.dimension = layer_index, dimension


class EvalFailure(RuntimeError):
    """A candidate could not be scored (diverged, OOM, device fault, timeout).
    Turned into an ok=False record with fitness -inf; never kills the run."""

    def __init__(self, reason):
        RuntimeError.__init__(self, reason)
        self.reason = reason


class FormatError(ValueError):
    """On-disk container does not match its declared format."""

    def __init__(self, message, offset=None):
        ValueError.__init__(self, message)
        self.offset = offset


class ConfigError(ValueError):
    """Invalid run configuration."""


class ProtocolError(ValueError):
    """Malformed message on the worker transport."""


class NativeError(EvalFailure):
    """Failure reported by libmenndl_sm100 (status code kept for triage).

    ``sticky`` marks CUDA errors after which the device context is unusable;
    the scheduler stops issuing work to that GPU.
    """

    def __init__(self, status, message):
        EvalFailure.__init__(self, message)
        self.status = status
        self.sticky = status == CE_ECUDA and any(
            tok in message for tok in ("illegal", "misaligned", "launch failure", "unspecified"))


def status_to_exception(status, message):
    if status == CE_EINVAL:
        return ShapeError(message)
    return NativeError(status, message)
