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


def device_scratch(pd, nq, x_count=None, path="gray", device="cuda:0"):
    """Scratch for the device entry points: pd_scratch_bytes(N, x_count, path) — the diagonals
    of the X-mask range plus their non-finite flags — as a complex128 tensor."""
    import torch
    nbytes = pd.device.scratch_bytes(nq, 2**nq if x_count is None else x_count, path)
    return torch.empty((nbytes + 15) // 16, dtype=torch.complex128, device=device)


def same_values(a, b):
    """Equal as complex numbers (IEEE ==, so -0.0 == +0.0; SURVEY §7 signed zeros)."""
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and bool(np.all(a == b))


def same_or_both_nan(a, b):
    """Equal values with NaN in the same places (part by part; NaN payloads are not compared:
    x86 and CUDA generate different default NaNs). IEEE == otherwise, so -0.0 == +0.0."""
    a = np.asarray(a, dtype=complex)
    b = np.asarray(b, dtype=complex)
    return a.shape == b.shape and all(
        np.array_equal(p, q, equal_nan=True) for p, q in ((a.real, b.real), (a.imag, b.imag)))
