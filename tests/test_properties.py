"""Property-based checks (hypothesis) of the index algebra and of the oracle against the
reference compiled from its own sources, on randomly drawn sizes, indices and matrices.

CPU only: the package's host-side helpers (label/index/mask algebra, run offsets) need no GPU,
and the oracle port is compared with oracle/_ref when that was built in this container."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from conftest import same_values
from oracle import oracle as O

SETTINGS = settings(max_examples=60, deadline=None,
                    suppress_health_check=[HealthCheck.function_scoped_fixture])


def _digits(n: int, nq: int):
    return [(n >> (2 * t)) & 3 for t in range(nq)]


@SETTINGS
@given(st.integers(1, 20).flatmap(lambda nq: st.tuples(st.just(nq), st.integers(0, 4**nq - 1))))
def test_label_index_round_trip_and_masks(pd, args):
    nq, n = args
    label = pd.index_to_label(n, nq)
    assert len(label) == nq and pd.label_to_index(label, nq) == n
    d = _digits(n, nq)
    # digit 0 is the rightmost character (pauli.hpp:13-20)
    assert label == "".join("IXYZ"[d[t]] for t in reversed(range(nq)))
    x = pd.xy_mask(n, nq)
    assert x == sum(((d[t] in (1, 2)) << t) for t in range(nq))


@SETTINGS
@given(st.integers(0, 2**40))
def test_gray_code_and_flipped_bit(pd, k):
    assert pd.gray_code(k) == k ^ (k >> 1)
    # the bit that flips between g(k) and g(k+1) (bits.hpp:71-81)
    assert pd.gray_code(k) ^ pd.gray_code(k + 1) == 1 << pd.flipped_bit_index(k)


@SETTINGS
@given(st.integers(1, 12).flatmap(
    lambda nq: st.tuples(st.just(nq), st.integers(0, min(nq, 8)).flatmap(
        lambda p: st.tuples(st.just(p), st.integers(0, 2**p - 1), st.integers(0, 2**p - 1))))))
def test_run_offsets_match_tensor_numbers(pd, args):
    """run r of X-mask block g (p top bits) starts at the tensor number whose top digits come
    from x's top bits = g and z's top bits = r, low digits zero"""
    nq, (p, g, r) = args
    off = pd.device.run_offset(nq, p, g, r)
    x = g << (nq - p)
    z = r << (nq - p)
    assert off == int(O.xz_to_n(np.uint64(x), np.array([z], dtype=np.uint64), nq)[0])


@SETTINGS
@given(st.integers(1, 5), st.integers(0, 2**32 - 1), st.integers(1, 40))
def test_port_equals_compiled_reference(port, ref, nq, seed, count):
    """coeff_fast, coeff_slow and the full decomposition of the C restatement equal the
    reference's own compiled code bit for bit on random matrices and strings"""
    if ref is None:
        pytest.skip("oracle/_ref not built in this container")
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((2**nq, 2**nq)) + 1j * rng.standard_normal((2**nq, 2**nq))
    assert same_values(port.decompose(g, threads=1), ref.decompose(g, threads=1))
    ns = rng.integers(0, 4**nq, count).astype(np.uint64)
    assert same_values(port.coeff_batch(g, ns, threads=1), ref.coeff_batch(g, ns, threads=1))
    n = int(ns[0])
    assert same_values(np.array([port.coeff_slow(g, n)]), np.array([ref.coeff_slow(g, n)]))
