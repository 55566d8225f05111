import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)
GOLDEN = os.path.join(HERE, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def rel(a: float, b: float) -> float:
    """The reference suite's metric (pkg/tests/conftest.py:137-144)."""
    return abs(a - b) / max(1.0, abs(a), abs(b))


def max_rel(x, y) -> float:
    """Elementwise max of ``rel`` over arrays / scalars (vectorised)."""
    x = np.asarray(_host(x), dtype=np.float64)
    y = np.asarray(_host(y), dtype=np.float64)
    if x.size == 0 and y.size == 0:
        return 0.0
    x, y = np.broadcast_arrays(x, y)
    den = np.maximum(1.0, np.maximum(np.abs(x), np.abs(y)))
    d = np.abs(x - y) / den
    if np.isnan(d).any():
        return float("inf")
    return float(d.max())


def _host(v):
    if hasattr(v, "detach"):
        return v.detach().cpu().double().numpy()
    if hasattr(v, "data") and isinstance(getattr(v, "data"), np.ndarray):
        return v.data
    return v


def decode(v):
    """Fixture value -> float or float64 ndarray."""
    if isinstance(v, dict):
        return np.array(v["data"], dtype=np.float64).reshape(v["shape"])
    return float(v)


@pytest.fixture(scope="session")
def golden_fused():
    with open(os.path.join(GOLDEN, "fused.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def fused_module():
    from fused_src import FUSED_SRC
    from paper_1811_01457_b200.irtext import parse_ir

    return parse_ir(FUSED_SRC)


def load_npz(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
