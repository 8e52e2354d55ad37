"""Shared fixtures. `-m gpu` tests need a B200 (sm_100); everything else runs on CPU."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_vectors.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (B200)")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O
    return O.port()


@pytest.fixture(scope="session")
def ref():
    """The reference's own compiled library (oracle/_ref), or skip when absent."""
    from oracle import oracle as O
    r = O.reference()
    if r is None:
        pytest.skip("oracle/_ref/libpdref.so not built (needs /root/reference at build time)")
    return r


@pytest.fixture(scope="session")
def pd():
    import paper_2401_16378_b200 as pd
    return pd


@pytest.fixture(scope="session")
def cuda(pd):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch.device("cuda:0")


def normal_matrix(rng, nq):
    """proj/tests/python/test_smoke.py:32-34 construction."""
    d = 2**nq
    return rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))


def same_values(a, b):
    """Equal as complex numbers (IEEE ==, so -0.0 == +0.0; SURVEY §7 signed zeros)."""
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and bool(np.all(a == b))
