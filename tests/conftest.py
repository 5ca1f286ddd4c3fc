import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O


@pytest.fixture(scope="session")
def ref_pristine():
    from oracle import oracle as O

    mod = O.ref_kernels("pristine")
    if mod is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    return mod


@pytest.fixture(scope="session")
def ref_corrected():
    from oracle import oracle as O

    mod = O.ref_kernels("corrected")
    if mod is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    return mod


@pytest.fixture(scope="session")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test on a box without CUDA")
    from paper_1705_01263_b200 import _abi

    return _abi.lib()
