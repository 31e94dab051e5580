"""Exception hierarchy of the drop-in surface.

Mirrors the reference's error types (``pkg/src/smmconv/errors.py:4-29``) so
callers that catch ``GeometryError`` / ``ShapeMismatchError`` keep working
unchanged.  Native (C-ABI) status codes are mapped onto these types by
``_native.raise_for_status``; CUDA failures surface as ``DeviceError`` — there
is never a silent CPU fallback.
"""

__all__ = [
    "SmmConvError",
    "GeometryError",
    "ShapeMismatchError",
    "BackendUnsupportedError",
    "ConfigError",
    "ChecksumMismatchError",
    "DeviceError",
]


class SmmConvError(Exception):
    """Root of every error raised by this package."""


class GeometryError(SmmConvError, ValueError):
    """Invalid convolution parameters (non-int, non-positive, empty output)."""


class ShapeMismatchError(SmmConvError, ValueError):
    """A tensor's shape, dtype, contiguity or device is not what the op needs."""


class BackendUnsupportedError(SmmConvError):
    """Valid geometry that the selected kernel variant does not implement."""


class ConfigError(SmmConvError, ValueError):
    """Malformed configuration."""


class ChecksumMismatchError(SmmConvError, RuntimeError):
    """Two implementations disagreed beyond the stated tolerance."""


class DeviceError(SmmConvError, RuntimeError):
    """A CUDA call failed, or the native library / GPU is unavailable."""
