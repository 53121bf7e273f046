"""Shared fixtures.  `-m gpu` tests need a B200 (they call the CUDA library
through the C ABI); everything else runs on CPU."""

from __future__ import annotations

import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: full-size BASELINE configurations")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name: str):
        if name not in cache:
            with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
                cache[name] = {k: z[k] for k in z.files}
        return cache[name]

    return load


@pytest.fixture(scope="session")
def sensitivity():
    from paper_1706_07263_b200 import fixtures

    return fixtures.default_sensitivity()


@pytest.fixture(scope="session")
def basis():
    from paper_1706_07263_b200 import fixtures

    return fixtures.default_basis()


@pytest.fixture()
def rng():
    return np.random.default_rng(20240817)


@pytest.fixture(scope="session")
def cuda():
    """The CUDA device the gpu tests run on (fails loudly if absent)."""
    import torch

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_1706_07263_b200 import _native

    _native.load()
    return torch.device("cuda", 0)
