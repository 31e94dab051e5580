"""Deterministic host fills used by the drop-in estimator.

``Conv2D.fit`` without explicit weights draws them from the reference's fixed
splitmix64 stream (``pkg/src/smmconv/tensors.py:43-62``), so the same ``seed``
must give bit-identical weights here; ``tests/test_host.py`` pins the stream
against the reference's golden head.  BASELINE synthetic inputs
(``synthetic_layer``) use numpy's PCG64 instead.
"""

import numpy as np

__all__ = ["fill_deterministic", "random_tensor", "synthetic_layer"]

_INC = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def fill_deterministic(out, seed):
    """Element i <- top 24 bits of splitmix64(seed + (i+1)*golden) * 2**-24."""
    count = out.size
    with np.errstate(over="ignore"):
        z = (np.arange(1, count + 1, dtype=np.uint64) * _INC
             + np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    vals = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / (1 << 24))
    out.reshape(-1)[:] = vals
    return out


def random_tensor(shape, seed):
    return fill_deterministic(np.empty(shape, dtype=np.float32), seed)


def synthetic_layer(geom, batch, seed):
    """BASELINE.json inputs: x ~ U[-1,1), W ~ N(0, sqrt(2/(c_i*k_h*k_w))) OIHW."""
    rng = np.random.default_rng(seed)
    x = rng.random((batch,) + geom.input_shape, dtype=np.float32)
    x *= np.float32(2.0)
    x -= np.float32(1.0)
    std = np.float32(np.sqrt(2.0 / (geom.in_channels * geom.k_h * geom.k_w)))
    w = rng.standard_normal(geom.weights_shape, dtype=np.float32)
    w *= std
    return x, w
