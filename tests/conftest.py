"""Shared fixtures: golden vectors (produced by the reference itself), the CPU
oracle (test infrastructure), and the ``gpu`` marker."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden" / "smm_golden.npz"

try:  # reference tests use hypothesis with a 'kernels' profile; mirror it
    from hypothesis import HealthCheck, settings
    settings.register_profile("kernels", deadline=None, max_examples=25,
                              suppress_health_check=[HealthCheck.too_slow])
    settings.load_profile("kernels")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class GoldenCase:
    def __init__(self, data, entry):
        from paper_2411_15659_b200 import ConvGeometry
        self.name = entry["name"]
        self.kind = entry["kind"]
        self.n = entry["n"]
        self.geom = ConvGeometry(*entry["geom"])
        self._data = data

    def __getattr__(self, item):
        key = f"{self.name}__{item}"
        if key in self._data.files:
            return self._data[key]
        raise AttributeError(item)

    def __repr__(self):
        return f"GoldenCase({self.name})"


def _load_golden():
    data = np.load(GOLDEN)
    manifest = json.loads(str(data["manifest"]))
    return data, manifest


_DATA, _MANIFEST = _load_golden()
GOLDEN_CASES = [GoldenCase(_DATA, e) for e in _MANIFEST["cases"] if e["kind"] != "slices"]
GOLDEN_SLICES = [e for e in _MANIFEST["cases"] if e["kind"] == "slices"][0]


@pytest.fixture(scope="session")
def golden_data():
    return _DATA


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def sample_geometry(rng, max_channels=4, max_hw=12, kernels=(1, 3, 5),
                    strides=(1, 2), paddings=(0, 1)):
    """Random small geometry, same grid as the reference's conftest.py:52-70."""
    from paper_2411_15659_b200 import ConvGeometry
    while True:
        kw = dict(in_channels=int(rng.integers(1, max_channels + 1)),
                  out_channels=int(rng.integers(1, max_channels + 1)),
                  in_h=int(rng.integers(4, max_hw + 1)), in_w=int(rng.integers(4, max_hw + 1)),
                  k_h=int(rng.choice(kernels)), k_w=int(rng.choice(kernels)),
                  stride_h=int(rng.choice(strides)), stride_w=int(rng.choice(strides)),
                  pad_h=int(rng.choice(paddings)), pad_w=int(rng.choice(paddings)))
        if kw["k_h"] <= kw["in_h"] + 2 * kw["pad_h"] and kw["k_w"] <= kw["in_w"] + 2 * kw["pad_w"]:
            return ConvGeometry(**kw)
