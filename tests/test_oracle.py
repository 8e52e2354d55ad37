"""Pin the CPU oracle (oracle/pd_oracle.c) before trusting it as the GPU checker.

Sources of truth, in order: the reference's own known-answer tests
(proj/tests/test_decompose.cpp:69-105, proj/tests/python/test_smoke.py:57-65), golden vectors
produced by the reference itself (tests/golden/make_golden.py), and — where it was built in
this container — the reference library compiled from its own sources (oracle/_ref).
"""
import numpy as np
import pytest

from conftest import normal_matrix, same_or_both_nan, same_values
from oracle import oracle as O


def test_kat_single_qubit_exact(port, golden):
    # test_decompose.cpp:69-77: exact equality
    g = np.array([[1, 2], [3, 4]], dtype=complex)
    got = port.decompose(g, threads=1)
    assert list(got) == [2.5, 2.5, -0.5j, -1.5]
    assert same_values(got, golden["kat_coeffs"])
    assert port.coeff_slow(g, 3) == -1.5


def test_identity_lone_unit(port):
    # test_decompose.cpp:79-86
    for nq in (1, 2, 3):
        d = port.decompose(np.eye(2**nq, dtype=complex))
        assert d[0] == 1.0 and np.all(d[1:] == 0)


def test_hadamard_square(port):
    # test_decompose.cpp:88-105: XX = XZ = ZX = ZZ = 0.5
    h = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    d = port.decompose(np.kron(h, h).astype(complex))
    for n in range(16):
        lab = "IXYZ"[n >> 2] + "IXYZ"[n & 3]
        want = 0.5 if lab in ("XX", "XZ", "ZX", "ZZ") else 0.0
        assert abs(d[n] - want) < 1e-15


@pytest.mark.parametrize("nq", range(1, 7))
def test_normal_matrices_match_reference_bitwise(port, golden, nq):
    g = golden[f"normal{nq}_matrix"]
    np.testing.assert_array_equal(g, normal_matrix(np.random.default_rng(1234 + nq), nq))
    got = port.decompose(g)
    assert same_values(got, golden[f"normal{nq}_coeffs"])
    assert same_values(got, golden[f"normal{nq}_serial"])


@pytest.mark.parametrize("nq", range(1, 7))
def test_reference_generator_and_coefficients(port, golden, nq):
    seed = int(golden[f"unif{nq}_seed"])
    assert port.matrix_seed(20260823, nq, 0) == seed  # bench.cpp:42-46
    g = port.random_matrix(nq, seed)  # bench.cpp:48-58
    assert np.array_equal(g.view(np.uint64), golden[f"unif{nq}_matrix"].view(np.uint64))
    assert same_values(port.decompose(g), golden[f"unif{nq}_coeffs"])


def splitmix_at(seed: int, j: np.ndarray) -> np.ndarray:
    """Draw j of the splitmix64 stream (the jump-ahead the device generator K5 uses)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (j.astype(np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def unit_interval(bits: np.ndarray) -> np.ndarray:
    return (bits >> np.uint64(11)).astype(np.float64) * 2.0**-53 * 2.0 - 1.0


def test_generator_jump_ahead_matches_reference_at_n14(golden):
    # the device generator evaluates draw j directly; pin that formula on the reference's
    # own N=14 stream (head, tail and 4096 scattered elements)
    seed = int(golden["unif14_seed"])
    for k, want in ((np.arange(4096), golden["unif14_head"]),
                    (np.arange(4**14 - 4096, 4**14), golden["unif14_tail"]),
                    (golden["unif14_idx"].astype(np.int64), golden["unif14_at_idx"])):
        k = np.asarray(k, dtype=np.uint64)
        re = unit_interval(splitmix_at(seed, 2 * k))
        im = unit_interval(splitmix_at(seed, 2 * k + np.uint64(1)))
        got = re + 1j * im
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_hermitian_real_coefficients(port, golden):
    got = port.decompose(golden["herm4_matrix"])
    assert same_values(got, golden["herm4_coeffs"])
    assert np.max(np.abs(got.imag)) <= 1e-12


def test_batched_strings(port, golden):
    got = port.coeff_batch(golden["batch8_matrix"], golden["batch8_ns"])
    assert same_values(got, golden["batch8_coeffs"])


def test_real_input_y_parity_exact_zero(port):
    # test_decompose.cpp:219-232
    g = port.random_matrix(3, 55).real.astype(complex)
    d = port.decompose(g)
    for n in range(64):
        ys = sum(((n >> (2 * t)) & 3) == 2 for t in range(3))
        assert (d[n].imag if ys % 2 == 0 else d[n].real) == 0.0


def test_recompose_round_trip(port):
    for nq in range(1, 5):
        g = port.random_matrix(nq, 4000 + nq)
        np.testing.assert_allclose(port.recompose(port.decompose(g)), g, rtol=0, atol=1e-12)


def test_index_algebra(port):
    # n(x, z) = spread(x ^ z) | spread(z) << 1 inverts xy_mask / z-mask
    nq = 5
    z = np.arange(32, dtype=np.uint64)
    for x in (0, 1, 7, 22, 31):
        ns = O.xz_to_n(np.uint64(x), z, nq)
        assert sorted(ns.tolist()) == sorted(set(ns.tolist()))
        assert all(port.xy_mask(int(n), nq) == x for n in ns)
    # every n appears for exactly one (x, z)
    allns = np.concatenate([O.xz_to_n(np.uint64(x), z, nq) for x in range(32)])
    assert np.array_equal(np.sort(allns), np.arange(4**nq, dtype=np.uint64))


def test_port_matches_compiled_reference_bitwise(port, ref):
    rng = np.random.default_rng(5)
    for nq in range(1, 8):
        g = normal_matrix(rng, nq)
        a = ref.decompose(g)
        b = port.decompose(g)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
        ns = rng.integers(0, 4**nq, 64).astype(np.uint64)
        assert np.array_equal(ref.coeff_batch(g, ns, threads=2).view(np.uint64),
                              port.coeff_batch(g, ns, threads=2).view(np.uint64))
        for n in (0, 4**nq - 1):
            assert ref.coeff_slow(g, n) == port.coeff_slow(g, n)
        if nq <= 5:
            assert np.allclose(ref.recompose(a), port.recompose(b), atol=1e-12)


def test_compiled_reference_matches_its_own_golden(ref, golden):
    seed = int(golden["unif14_seed"])
    h = ref.random_matrix_handle(10, 77)
    assert h.nq == 10
    g6 = golden["unif6_matrix"]
    assert same_values(ref.decompose(g6), golden["unif6_coeffs"])
    assert same_values(ref.coeff_batch(golden["batch8_matrix"], golden["batch8_ns"]),
                       golden["batch8_coeffs"])
    assert ref.matrix_seed(20260823, 14, 0) == seed


def test_nonfinite_elements_match_reference_golden(port, golden):
    """Non-finite elements follow the reference's complex product (decompose.cpp:40): 0 * inf
    is NaN in the other component, and libgcc's Annex G recovery when both parts are NaN.
    [[1, inf], [3, 4]] -> [2.5, inf + nan i, nan + inf i, -1.5]."""
    got = port.decompose(golden["nfkat_matrix"], threads=1)
    assert same_or_both_nan(got, golden["nfkat_coeffs"])
    assert np.isnan(got[1].imag) and got[1].real == np.inf
    assert np.isnan(got[2].real) and got[2].imag == np.inf
    k = 0
    while f"nf{k}_matrix" in golden:
        g = golden[f"nf{k}_matrix"]
        want = golden[f"nf{k}_coeffs"]
        assert same_or_both_nan(port.decompose(g), want), k
        assert same_or_both_nan(want, golden[f"nf{k}_serial"]), k
        slow = golden[f"nf{k}_slow"]
        assert same_or_both_nan([port.coeff_slow(g, n) for n in range(slow.size)], slow), k
        assert same_or_both_nan(port.coeff_batch(g, np.arange(want.size, dtype=np.uint64)), want)
        assert same_or_both_nan(port.recompose(want), golden[f"nf{k}_recomposed"]), k
        k += 1
    assert k >= 8


def test_nonfinite_elements_match_compiled_reference(port, ref):
    """Every special value (+-0, +-inf, NaN, in either part) at every position of 2x2 matrices,
    and random sprinkles up to N=5, against the reference library itself."""
    specials = [0.0, -0.0, 1.5, -2.0, np.inf, -np.inf, np.nan]
    rng = np.random.default_rng(41)
    for pos in range(4):
        for re in specials:
            for im in specials:
                g = normal_matrix(rng, 1)
                g.real.flat[pos] = re
                g.imag.flat[pos] = im
                a = ref.decompose(g, threads=1)
                assert same_or_both_nan(port.decompose(g, threads=1), a), (pos, re, im)
                for n in range(4):
                    assert same_or_both_nan(port.coeff_slow(g, n), ref.coeff_slow(g, n))
                assert same_or_both_nan(port.recompose(a), ref.recompose(a))
    for trial in range(200):
        nq = int(rng.integers(1, 6))
        g = normal_matrix(rng, nq)
        for _ in range(int(rng.integers(1, 4))):
            part = g.real if rng.random() < 0.5 else g.imag
            part.flat[int(rng.integers(0, 4**nq))] = rng.choice(specials)
        a = ref.decompose(g)
        assert same_or_both_nan(port.decompose(g), a), (trial, nq)
        assert same_or_both_nan(port.recompose(a), ref.recompose(a)), (trial, nq)
