"""B200-native (sm_100a) SMM-Conv: forward NCHW convolution by scalar-matrix
accumulation with zero packing (arxiv 2411.15659), behind the reference
``smmconv`` package's own entry points.

Hot-path names mirror ``pkg/src/smmconv/__init__.py:46-79`` (the ★ subset of
SURVEY §2.1); the compute is the CUDA library ``lib/libsmmc.so`` (C ABI:
``include/smmc.h``).  There is no CPU fallback.
"""

from .errors import (BackendUnsupportedError, ChecksumMismatchError,
                     ConfigError, DeviceError, GeometryError,
                     ShapeMismatchError, SmmConvError)
from .geometry import ConvGeometry, output_shape
from .smm import (extract_slice, gpu_workspace_bytes, repack_weights,
                  scalar_matrix_fma, shifted_view, smm_conv_batched,
                  smm_conv_parallel, smm_conv_single, smm_workspace_elements,
                  unpack_weights)
from .tensors import fill_deterministic, random_tensor

__version__ = "0.1.0"


def __getattr__(name):
    # sklearn is imported lazily so the core path does not require it.
    if name == "Conv2D":
        from .estimator import Conv2D
        return Conv2D
    raise AttributeError(name)


__all__ = [
    "BackendUnsupportedError",
    "ChecksumMismatchError",
    "ConfigError",
    "Conv2D",
    "ConvGeometry",
    "DeviceError",
    "GeometryError",
    "ShapeMismatchError",
    "SmmConvError",
    "extract_slice",
    "fill_deterministic",
    "gpu_workspace_bytes",
    "output_shape",
    "random_tensor",
    "repack_weights",
    "scalar_matrix_fma",
    "shifted_view",
    "smm_conv_batched",
    "smm_conv_parallel",
    "smm_conv_single",
    "smm_workspace_elements",
    "unpack_weights",
]
