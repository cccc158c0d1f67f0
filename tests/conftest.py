import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: full-size BASELINE configurations")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.orc()
    return oracle


@pytest.fixture(scope="session")
def ref_lib():
    import oracle
    if not oracle.ref_available():
        pytest.skip("reference library oracle/_ref/libfea_ref.so not available")
    return oracle


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2012_00585_b200 as fea
    fea._native.lib()  # fail loudly if the native library is missing
    return fea
