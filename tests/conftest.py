import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def reflib():
    import oracle

    oracle.build_ref()
    if not oracle.ref_available():
        pytest.skip("reference library (oracle/_ref) not built")
    return oracle.RefLib()


@pytest.fixture(scope="session")
def gpu():
    """The product library on cuda:0; fails loudly (no fallback) when absent on a GPU box."""
    from paper_2202_07569_b200 import build

    build.build()
    if not cuda_available():
        pytest.skip("no CUDA device")
    from paper_2202_07569_b200 import load_library

    return load_library()


def small_params(N=1024, L=3, bits=36, t=12289):
    from paper_2202_07569_b200 import configs

    return N, configs.custom_chain(N, L, bits), t


def rng(seed=0):
    return np.random.default_rng(seed)
