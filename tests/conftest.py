from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "fullsize: BASELINE configs at full size (GPU, minutes)")
    config.addinivalue_line("markers", "reference: needs the reference package (build container only)")


def have_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    gpu = have_gpu()
    for item in items:
        if "gpu" in item.keywords and not gpu:
            item.add_marker(pytest.mark.skip(reason="no CUDA device"))


@pytest.fixture(scope="session")
def ref():
    """The reference `pipal` package (only importable in the build container)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference package not present (GPU box)")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    import pipal  # noqa: F401
    from pipal import baselines, relaxed, runtime, strong

    class R:
        pass

    r = R()
    r.baselines, r.relaxed, r.runtime, r.strong = baselines, relaxed, runtime, strong
    return r


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle

    oracle.build()
    return oracle


def golden(name: str):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


def rand_words(seed, n, hi=None):
    rng = np.random.default_rng(seed)
    if hi is None:
        return rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
    return rng.integers(0, hi, size=n, dtype=np.uint64)
