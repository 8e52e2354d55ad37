"""GPU parity on non-finite elements.

The reference multiplies every term as std::complex<double> (lambda.value() * a[...],
proj/src/decompose.cpp:40): 0 * inf is NaN in the other component, and libgcc's C99 Annex G
recovery applies when both parts are NaN. So [[1, inf], [3, 4]] decomposes to
[2.5, inf + nan i, nan + inf i, -1.5], not to the add/swap result (inf + 0i, 0 + inf i).
Every path must reproduce that: the fast kernels flag X-masks whose diagonal holds an inf or NaN
(K1, the WHT's pass 1) and pd_nonfinite.cu recomputes them with the reference's products; the
single-string walks redo a non-finite sum the same way. Compared NaN-aware (NaN in the same
places, infinities with their signs, IEEE == elsewhere) against the reference's own outputs
(tests/golden) and the oracle port, which is pinned to the compiled reference on these inputs
(tests/test_oracle.py).
"""
import numpy as np
import pytest

from conftest import device_scratch, normal_matrix, same_or_both_nan
from oracle import oracle as O

pytestmark = pytest.mark.gpu

SPECIALS = np.array([np.inf, -np.inf, np.nan])


def sprinkle(rng, g, count):
    """put `count` specials into random parts of g (in place); returns the X-masks they hit"""
    nq = g.shape[0].bit_length() - 1
    xs = set()
    for _ in range(count):
        i = int(rng.integers(0, g.size))
        part = g.real if rng.random() < 0.5 else g.imag
        part.flat[i] = rng.choice(SPECIALS)
        row, col = divmod(i, 2**nq)
        xs.add(row ^ col)
    return sorted(xs)


def matches(got, want, path):
    """Gray / naive: every value (NaN-aware, IEEE ==). WHT: the X-masks with a non-finite
    element take the reference's products, so every non-finite coefficient is exact there; the
    finite ones are within the north-star tolerance 1e-11 * max|c| (different summation order)."""
    if path != "wht":
        return same_or_both_nan(got, want)
    got = np.asarray(got)
    want = np.asarray(want)
    fin = np.isfinite(want)
    if not same_or_both_nan(got[~fin], want[~fin]) or not np.all(np.isfinite(got[fin])):
        return False
    if not fin.any():
        return True
    return np.max(np.abs(got[fin] - want[fin])) <= 1e-11 * max(np.max(np.abs(want[fin])), 1e-300)


def xmask_ns(nq, xs):
    return O.xmask_sample_indices(nq, xs)


def test_kat_nonfinite_every_path(pd, cuda, golden):
    g = golden["nfkat_matrix"]
    want = golden["nfkat_coeffs"]
    for path in ("gray", "wht", "naive"):
        assert matches(pd.decompose(g, path=path), want, path), path
    assert same_or_both_nan(pd.decompose(g, serial=True), want)
    for n in range(4):
        assert same_or_both_nan(pd.coefficient(g, n), want[n])
        assert same_or_both_nan(pd.coefficient(g, n, slow=True), want[n])
    assert same_or_both_nan(pd.coefficients(g, np.arange(4, dtype=np.uint64)), want)


def test_golden_nonfinite_matrices(pd, cuda, golden):
    k = 0
    while f"nf{k}_matrix" in golden:
        g = golden[f"nf{k}_matrix"]
        want = golden[f"nf{k}_coeffs"]
        for path in ("gray", "wht", "naive"):
            assert matches(pd.decompose(g, path=path), want, path), (k, path)
        assert same_or_both_nan(pd.decompose(g, serial=True), want), k
        slow = golden[f"nf{k}_slow"]
        for n in range(slow.size):
            assert same_or_both_nan(pd.coefficient(g, n, slow=True), slow[n]), (k, n)
            assert same_or_both_nan(pd.coefficient(g, n), want[n]), (k, n)
        ns = np.arange(want.size, dtype=np.uint64)
        assert same_or_both_nan(pd.coefficients(g, ns), want), k
        k += 1
    assert k >= 8


def test_oracle_coefficient_nonfinite(pd, cuda, ref):
    """oracle_coeff_kron (decompose.cpp:176-203) multiplies every P_n entry, zeros included"""
    rng = np.random.default_rng(17)
    for nq in (1, 2, 3):
        g = normal_matrix(rng, nq)
        sprinkle(rng, g, 2)
        for n in range(min(4**nq, 20)):
            assert same_or_both_nan(pd.oracle_coefficient(g, n), ref.oracle_kron(g, n)), (nq, n)


@pytest.mark.parametrize("nq", [7, 8, 9, 10, 11])
def test_full_decomposition_nonfinite_all_paths(pd, cuda, port, nq):
    """N=7..11: K2 / K2s, the fused WHT, the host pipeline (N >= 10) — whole arrays"""
    rng = np.random.default_rng(900 + nq)
    g = normal_matrix(rng, nq)
    xs = sprinkle(rng, g, 3)
    want = port.decompose(g)
    for path in ("gray", "wht", "naive"):
        got = pd.decompose(g, path=path)
        assert matches(got, want, path), (nq, path, xs)
    assert np.isnan(want).any()


@pytest.mark.parametrize("nq", [12, 13, 14])
def test_large_nonfinite_host_and_device_paths(pd, cuda, port, nq):
    """N=12..14 (the segmented host pipeline, K2s-c at N >= 13, the chunked WHT): the flagged
    X-masks in full against the oracle, a seeded sample of the others, and the device path equal
    to the host path"""
    import torch
    rng = np.random.default_rng(1200 + nq)
    g = port.random_matrix(nq, 77 + nq)
    xs = sprinkle(rng, g, 2)
    ns_bad = xmask_ns(nq, xs)
    want_bad = port.coeff_batch(g, ns_bad)
    ns_ok = np.sort(rng.choice(4**nq, 8192, replace=False)).astype(np.uint64)
    want_ok = port.coeff_batch(g, ns_ok)
    gd = torch.from_numpy(g).to(cuda)
    out = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    scratch = device_scratch(pd, nq, path="wht")
    for path in ("gray", "wht"):
        host = pd.decompose(g, path=path)
        assert matches(host[ns_bad.astype(np.int64)], want_bad, path), (nq, path)
        assert matches(host[ns_ok.astype(np.int64)], want_ok, path), (nq, path)
        pd.device.decompose(nq, gd.data_ptr(), out.data_ptr(), scratch.data_ptr(), path, 0)
        torch.cuda.synchronize()
        dev = out.cpu().numpy()
        assert matches(dev[ns_bad.astype(np.int64)], want_bad, path), (nq, path)
        if path == "gray":
            assert same_or_both_nan(dev, host)
        del host, dev


def test_sharded_layouts_nonfinite(pd, cuda, port):
    """the multi-GPU addressing (GLOBAL in place, RUNS packed) with flagged X-masks in every
    shard: the fixup stores through the same output map as K2 / the WHT"""
    import torch
    nq = 9
    rng = np.random.default_rng(9009)
    gh = normal_matrix(rng, nq)
    sprinkle(rng, gh, 6)
    want = port.decompose(gh)
    g = torch.from_numpy(gh).to(cuda)
    for p in (1, 2, 3):
        xc = 2 ** (nq - p)
        diag = device_scratch(pd, nq, max(xc, 32))
        packed = torch.empty(4**nq >> p, dtype=torch.complex128, device=cuda)
        rl = 4 ** (nq - p)
        for path in ("gray", "wht"):
            out = torch.zeros(4**nq, dtype=torch.complex128, device=cuda)
            out_runs = torch.zeros_like(out)
            for shard in range(2**p):
                pd.device.shard_coeffs(nq, g.data_ptr(), shard * xc, xc, p, out.data_ptr(),
                                       "global", diag.data_ptr(), path, 0)
                pd.device.shard_coeffs(nq, g.data_ptr(), shard * xc, xc, p, packed.data_ptr(),
                                       "runs", diag.data_ptr(), path, 0)
                for r in range(2**p):
                    o = pd.device.run_offset(nq, p, shard, r)
                    out_runs[o:o + rl] = packed[r * rl:(r + 1) * rl]
            torch.cuda.synchronize()
            for o in (out, out_runs):
                assert matches(o.cpu().numpy(), want, path), (p, path)
            # K1 + K2 through the diagonal entry points
            if path == "gray":
                out2 = torch.zeros_like(out)
                for shard in range(2**p):
                    pd.device.diag_gather(nq, g.data_ptr(), shard * xc, xc, diag.data_ptr(), 0)
                    pd.device.xmask_coeffs(nq, diag.data_ptr(), shard * xc, xc, p, out2.data_ptr(),
                                           "global", "gray", 0)
                torch.cuda.synchronize()
                assert same_or_both_nan(out2.cpu().numpy(), want), p


def test_batched_and_single_strings_nonfinite(pd, cuda, port):
    """K3b (grouped strings, N=10 BASELINE configs[1] shape), K3 (slow), the one-string walk at
    N=14 and the sparse-diagonal batch path, on matrices with infinities and NaNs"""
    rng = np.random.default_rng(1010)
    g = normal_matrix(rng, 10)
    xs = sprinkle(rng, g, 20)
    ns = rng.integers(0, 4**10, 65536).astype(np.uint64)
    ns[:4096] = xmask_ns(10, xs[:4])[:4096]
    want = port.coeff_batch(g, ns)
    assert not np.all(np.isfinite(want))
    assert same_or_both_nan(pd.coefficients(g, ns), want)
    for n in ns[:8]:
        assert same_or_both_nan(pd.coefficient(g, int(n), slow=True), want[list(ns).index(n)])
    g14 = port.random_matrix(14, 1414)
    xs = sprinkle(rng, g14, 1)
    ns14 = xmask_ns(14, xs)[::4099][:4]
    w14 = port.coeff_batch(g14, ns14)
    for n, w in zip(ns14, w14):
        assert same_or_both_nan(pd.coefficient(g14, int(n)), w)
    assert same_or_both_nan(pd.coefficients(g14, ns14), w14)   # few X-masks: gathered diagonals


def test_wht_in_place_passes_nonfinite_n13(pd, cuda, port):
    """pd_xmask_coeffs_device on the WHT path at N > 12 rewrites the diagonals in place, so the
    non-finite X-masks are found (nonfinite_scan) and recomputed before the passes, which skip
    them; the rest within the tolerance"""
    import torch
    nq, xc, x0 = 13, 16, 48
    rng = np.random.default_rng(1313)
    gh = port.random_matrix(nq, 1313)
    dim = 2**nq
    for x in (x0 + 3, x0 + 10):   # an inf and a NaN on two diagonals of the range
        i = int(rng.integers(0, dim))
        gh[i ^ x, i] = complex(np.inf, gh[i ^ x, i].imag) if x == x0 + 3 else complex(1.0, np.nan)
    g = torch.from_numpy(gh).to(cuda)
    diag = device_scratch(pd, nq, xc)
    out = torch.zeros(4**nq, dtype=torch.complex128, device=cuda)
    pd.device.diag_gather(nq, g.data_ptr(), x0, xc, diag.data_ptr(), 0)
    pd.device.xmask_coeffs(nq, diag.data_ptr(), x0, xc, 0, out.data_ptr(), "global", "wht", 0)
    torch.cuda.synchronize()
    ns = xmask_ns(nq, list(range(x0, x0 + xc)))
    want = port.coeff_batch(gh, ns)
    got = out[torch.from_numpy(ns.astype(np.int64)).to(cuda)].cpu().numpy()
    assert matches(got, want, "wht")
    assert (~np.isfinite(want)).sum() >= dim
