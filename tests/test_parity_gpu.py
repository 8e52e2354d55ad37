"""GPU parity: the CUDA path against the oracle and the reference's own golden vectors.

Bar (BASELINE.json north_star): max|dc| <= 1e-11 max|c| in complex128 and bit-exact index
and phase assignment. The Gray path (K1+K2) and the naive walk (K0/K3) sum each coefficient
in the reference's exact order, so they are held to IEEE equality (== on values; the sign of
an exact zero may differ). The WHT path is held to the tolerance.
"""
import numpy as np
import pytest

from conftest import ROOT, device_scratch, normal_matrix, same_values
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-11  # north_star: max|dc| <= 1e-11 * max|c|


def rel_err(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_kat_exact(pd, cuda):
    g = np.array([[1, 2], [3, 4]], dtype=complex)
    assert pd.coefficient(g, "I") == 2.5
    assert pd.coefficient(g, "X") == 2.5
    assert pd.coefficient(g, "Y") == -0.5j
    assert pd.coefficient(g, "Z") == -1.5
    assert pd.coefficient(g, 3) == -1.5
    assert pd.coefficient(g, 3, slow=True) == pd.coefficient(g, 3)
    assert pd.oracle_coefficient(g, "Z") == pytest.approx(-1.5)
    for path in ("gray", "naive", "wht"):
        assert list(pd.decompose(g, path=path)) == [2.5, 2.5, -0.5j, -1.5]


def test_identity_and_hadamard(pd, cuda):
    for nq in (1, 2, 3):
        d = pd.decompose(np.eye(2**nq, dtype=complex))
        assert d[0] == 1.0 and np.all(d[1:] == 0)
    h = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    d = pd.decompose(np.kron(h, h).astype(complex))
    for n in range(16):
        lab = pd.index_to_label(n, 2)
        want = 0.5 if lab in ("XX", "XZ", "ZX", "ZZ") else 0.0
        assert abs(d[n] - want) < 1e-15


@pytest.mark.parametrize("nq", range(1, 7))
@pytest.mark.parametrize("path", ["gray", "naive"])
def test_reference_order_paths_equal_reference(pd, cuda, golden, nq, path):
    for key in (f"normal{nq}", f"unif{nq}"):
        got = pd.decompose(golden[f"{key}_matrix"], path=path)
        assert same_values(got, golden[f"{key}_coeffs"]), (key, path)


@pytest.mark.parametrize("nq", range(1, 7))
def test_wht_path_within_tolerance(pd, cuda, golden, nq):
    for key in (f"normal{nq}", f"unif{nq}"):
        got = pd.decompose(golden[f"{key}_matrix"], path="wht")
        assert rel_err(got, golden[f"{key}_coeffs"]) <= TOL


def test_slow_and_oracle_coefficients(pd, cuda, golden, port):
    g = golden["normal5_matrix"]
    c = golden["normal5_coeffs"]
    for n in (0, 1, 2, 3, 100, 511, 1023):
        assert pd.coefficient(g, n) == c[n]
        assert pd.coefficient(g, n, slow=True) == c[n]
        assert abs(pd.oracle_coefficient(g, n) - c[n]) <= 1e-12 * (1 + abs(c[n]))
    assert pd.coefficient(g, pd.index_to_label(777, 5)) == c[777]
    with pytest.raises(ValueError):
        pd.coefficient(g, 4**5)
    with pytest.raises(ValueError):
        pd.oracle_coefficient(np.eye(128, dtype=complex), 0)  # kOracleMaxQubits = 6


def test_batched_strings_golden(pd, cuda, golden):
    got = pd.coefficients(golden["batch8_matrix"], golden["batch8_ns"])
    assert same_values(got, golden["batch8_coeffs"])


def test_batched_strings_config2(pd, cuda, port):
    # BASELINE config 2: N=10 N(0,1) matrix, 65,536 uniformly drawn strings
    rng = np.random.default_rng(2)
    g = normal_matrix(rng, 10)
    ns = rng.integers(0, 4**10, 65536).astype(np.uint64)
    assert same_values(pd.coefficients(g, ns), port.coeff_batch(g, ns))


def test_hermitian_n10_config3(pd, cuda, port):
    # BASELINE config 3: G = (A + A^dagger)/2, 1,048,576 coefficients, imag ~ 0
    a = normal_matrix(np.random.default_rng(3), 10)
    g = (a + a.conj().T) / 2
    got = pd.decompose(g)
    assert np.max(np.abs(got.imag)) <= 1e-12
    assert same_values(got, port.decompose(g))


def test_full_n12_config4_sampled_bit_exact(pd, cuda, port):
    rng = np.random.default_rng(4)
    g = normal_matrix(rng, 12)
    got = pd.decompose(g)
    ns = rng.integers(0, 4**12, 65536).astype(np.uint64)
    want = port.coeff_batch(g, ns)
    assert same_values(got[ns.astype(np.int64)], want)
    # whole-array properties: Parseval ||G||_F^2 = 2^N sum |c|^2
    lhs = np.sum(np.abs(g) ** 2)
    rhs = 2**12 * np.sum(np.abs(got) ** 2)
    assert abs(lhs - rhs) <= 1e-10 * lhs
    assert rel_err(pd.decompose(g, path="wht"), got) <= TOL


@pytest.mark.parametrize("nq", [7, 8, 9, 10, 11, 13])
def test_wht_fused_sizes(pd, cuda, port, nq):
    g = normal_matrix(np.random.default_rng(700 + nq), nq)
    got = pd.decompose(g, path="wht")
    ns = np.random.default_rng(nq).integers(0, 4**nq, 4096).astype(np.uint64)
    assert rel_err(got[ns.astype(np.int64)], port.coeff_batch(g, ns)) <= TOL
    assert same_values(pd.decompose(g)[ns.astype(np.int64)], port.coeff_batch(g, ns))


@pytest.mark.parametrize("path", ["gray", "wht"])
@pytest.mark.parametrize("nq", [10, 12, 13])
def test_host_pipeline_matches_device_path(pd, cuda, nq, path):
    # the host pipelines (Gray: column segments; WHT: per-block tile uploads) against one
    # device-resident decomposition of the same matrix
    import torch
    g = normal_matrix(np.random.default_rng(1300 + nq), nq)
    gd = torch.from_numpy(g).to(cuda)
    out = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    scratch = device_scratch(pd, nq, path="wht")
    pd.device.decompose(nq, gd.data_ptr(), out.data_ptr(), scratch.data_ptr(), path, 0)
    torch.cuda.synchronize()
    assert np.array_equal(pd.decompose(g, path=path), out.cpu().numpy())


def test_integer_inputs_bit_exact_any_order(pd, cuda, port):
    # Gaussian-integer entries: every partial sum is exact, so all paths must agree bit for bit
    rng = np.random.default_rng(6)
    d = 2**11
    g = (rng.integers(-1000, 1000, (d, d)) + 1j * rng.integers(-1000, 1000, (d, d))).astype(complex)
    ref = port.decompose(g)
    for path in ("gray", "wht"):
        assert same_values(pd.decompose(g, path=path), ref), path


@pytest.mark.parametrize("nq", [8, 10])
def test_real_input_y_parity_exact_zero(pd, cuda, port, nq):
    """real G: coefficients with an even number of Y factors are real, odd ones imaginary, and
    the other part is an exact zero (N=10: K2s, whose chains carry region signs, N=8: K2)"""
    g = port.random_matrix(nq, 55).real.astype(complex)
    d = pd.decompose(g)
    n = np.arange(4**nq)
    ys = sum(((n >> (2 * t)) & 3) == 2 for t in range(nq))
    assert np.all(d.imag[ys % 2 == 0] == 0.0)
    assert np.all(d.real[ys % 2 == 1] == 0.0)
    assert same_values(d, port.decompose(g))


def test_structured_matrices_k2s_exact(pd, cuda, port):
    """K2s (N >= 9) on inputs whose sums cancel exactly: a Kronecker product of Paulis (one
    nonzero coefficient), a permutation matrix and a 0/1 band matrix — every coefficient equal
    to the reference walk's (IEEE ==)"""
    nq = 10
    P = [np.eye(2), np.array([[0, 1], [1, 0]]), np.array([[0, -1j], [1j, 0]]), np.diag([1, -1])]
    k = np.array([[1.0 + 0j]])
    for t in range(nq):
        k = np.kron(P[(3 * t + 1) % 4], k)
    perm = np.eye(2**nq)[np.random.default_rng(3).permutation(2**nq)].astype(complex)
    band = np.triu(np.tril(np.ones((2**nq, 2**nq)), 2), -1).astype(complex)
    for g in (k.astype(complex), perm, band):
        assert same_values(pd.decompose(g), port.decompose(g))


def test_recompose_round_trip(pd, cuda, port):
    rng = np.random.default_rng(99)
    for nq in range(1, 7):
        g = normal_matrix(rng, nq)
        np.testing.assert_allclose(pd.recompose(pd.decompose(g)), g, rtol=0, atol=1e-12)
    c = pd.decompose(normal_matrix(rng, 5))
    np.testing.assert_allclose(pd.recompose(c), port.recompose(c), rtol=0, atol=1e-12)


def _scatter_runs(pd, out, packed, nq, p, shard):
    """place a block's packed runs (PD_LAYOUT_RUNS) at their pd_run_offset in `out`"""
    rl = 4 ** (nq - p)
    for r in range(2**p):
        o = pd.device.run_offset(nq, p, shard, r)
        out[o:o + rl] = packed[r * rl:(r + 1) * rl]


def test_sharded_runs_assemble_full_array(pd, cuda):
    # the multi-GPU addressing, emulated shard by shard on one GPU (no collectives):
    # GLOBAL layout writes in place, RUNS layout packs each block (up to 2^8 blocks)
    import torch
    nq = 9
    g = torch.from_numpy(normal_matrix(np.random.default_rng(8), nq)).to(cuda)
    full = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    scratch = device_scratch(pd, nq, path="wht")
    pd.device.decompose(nq, g.data_ptr(), full.data_ptr(), scratch.data_ptr(), "gray", 0)
    for p in (1, 2, 3, 5, 8):
        xc = 2 ** (nq - p)
        diag = device_scratch(pd, nq, max(xc, 32))
        packed = torch.empty(4**nq >> p, dtype=torch.complex128, device=cuda)
        out = torch.zeros_like(full)
        out_runs = torch.zeros_like(full)
        for shard in range(2**p):
            pd.device.diag_gather(nq, g.data_ptr(), shard * xc, xc, diag.data_ptr(), 0)
            pd.device.xmask_coeffs(nq, diag.data_ptr(), shard * xc, xc, p, out.data_ptr(),
                                   "global", "gray", 0)
            pd.device.xmask_coeffs(nq, diag.data_ptr(), shard * xc, xc, p, packed.data_ptr(),
                                   "runs", "gray", 0)
            _scatter_runs(pd, out_runs, packed, nq, p, shard)
        torch.cuda.synchronize()
        assert torch.equal(out, full), p
        assert torch.equal(out_runs, full), p
        # the one-call shard entry point, both paths (WHT: fused two-pass from G when x_count >= 32)
        for path in ("gray", "wht"):
            out2 = torch.zeros_like(full)
            out3 = torch.zeros_like(full)
            for shard in range(2**p):
                pd.device.shard_coeffs(nq, g.data_ptr(), shard * xc, xc, p, out2.data_ptr(),
                                       "global", diag.data_ptr(), path, 0)
                pd.device.shard_coeffs(nq, g.data_ptr(), shard * xc, xc, p, packed.data_ptr(),
                                       "runs", diag.data_ptr(), path, 0)
                _scatter_runs(pd, out3, packed, nq, p, shard)
            torch.cuda.synchronize()
            for o in (out2, out3):
                if path == "gray":
                    assert torch.equal(o, full), (p, path)
                else:
                    err = float(torch.max(torch.abs(o - full)) / torch.max(torch.abs(full)))
                    assert err <= TOL, (p, err)


def test_xmask_range_validation(pd, cuda):
    import torch
    nq = 6
    g = torch.zeros((64, 64), dtype=torch.complex128, device=cuda)
    out = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    diag = device_scratch(pd, nq, 64)
    with pytest.raises(ValueError):   # spans two blocks of 2^(N-p)
        pd.device.shard_coeffs(nq, g.data_ptr(), 0, 64, 1, out.data_ptr(), "runs", diag.data_ptr())
    with pytest.raises(ValueError):   # run_bits > 8
        pd.device.shard_coeffs(nq, g.data_ptr(), 0, 1, 9, out.data_ptr(), "runs", diag.data_ptr())
    with pytest.raises(ValueError):   # misaligned range
        pd.device.shard_coeffs(nq, g.data_ptr(), 3, 2, 0, out.data_ptr(), "global", diag.data_ptr())
    with pytest.raises(ValueError):
        pd.device.shard_coeffs(nq, g.data_ptr(), 0, 64, 0, out.data_ptr(), "bogus", diag.data_ptr())


def test_n14_config5(pd, cuda, port, golden):
    """Full N=14 on the device from the reference's generator: 268,435,456 coefficients.

    Checked against the reference's own coeff_fast values (golden) and the oracle on a seeded
    sample of 65,536 coefficients, all bit-exact; plus Parseval over the whole array."""
    import torch
    nq = 14
    seed = int(golden["unif14_seed"])
    g = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=cuda)
    pd.device.random_matrix(nq, seed, g.data_ptr(), 0)
    flat = g.view(-1)
    idx = torch.from_numpy(golden["unif14_idx"].astype(np.int64)).to(cuda)
    assert torch.equal(flat[:4096].cpu(), torch.from_numpy(golden["unif14_head"]))
    assert torch.equal(flat[-4096:].cpu(), torch.from_numpy(golden["unif14_tail"]))
    assert torch.equal(flat[idx].cpu(), torch.from_numpy(golden["unif14_at_idx"]))
    out = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    scratch = device_scratch(pd, nq, path="wht")
    pd.device.decompose(nq, g.data_ptr(), out.data_ptr(), scratch.data_ptr(), "gray", 0)
    torch.cuda.synchronize()
    ns = golden["unif14_ns"].astype(np.int64)
    assert same_values(out[torch.from_numpy(ns).to(cuda)].cpu().numpy(), golden["unif14_ns_coeffs"])
    sample = np.sort(np.random.default_rng(14).choice(4**nq, 65536, replace=False))
    gh = g.cpu().numpy()
    want = port.coeff_batch(gh, sample.astype(np.uint64))
    got = out[torch.from_numpy(sample).to(cuda)].cpu().numpy()
    assert same_values(got, want)
    # the host-buffer path (segmented column upload + chained K2 segments + block D2H)
    # must reproduce the device-resident result exactly
    host = pd.decompose(gh)
    assert np.array_equal(host, out.cpu().numpy())
    del host
    fro = float(torch.sum(torch.abs(g) ** 2))
    par = float(2**nq * torch.sum(torch.abs(out) ** 2))
    assert abs(fro - par) <= 1e-10 * fro
    # WHT path agrees within the tolerance
    out2 = torch.empty_like(out)
    pd.device.decompose(nq, g.data_ptr(), out2.data_ptr(), scratch.data_ptr(), "wht", 0)
    torch.cuda.synchronize()
    err = float(torch.max(torch.abs(out2 - out)) / torch.max(torch.abs(out)))
    assert err <= TOL


def test_native_kernels_launched(pd, cuda):
    before = pd.launch_count()
    pd.decompose(np.eye(64, dtype=complex))
    assert pd.launch_count() >= before + 2  # K1 + K2


def test_n15_maximum_single_gpu_size(pd, cuda):
    """The largest full decomposition that fits one B200 with the scratch layout of
    pd_decompose_device (G, D and the coefficients: 3 x 16 GiB): N=15, 1,073,741,824
    coefficients. The Gray path (K1+K2) must equal the reference-order walk (K3, pinned to the
    oracle at N <= 14) on 65,536 seeded strings bit for bit; Parseval over the whole array;
    the WHT path within the tolerance."""
    import torch
    nq = 15
    torch.cuda.empty_cache()  # earlier tests' cached blocks
    free, _ = torch.cuda.mem_get_info()
    if free < 70 * 2**30:
        pytest.skip("needs ~64 GiB of free device memory")
    g = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=cuda)
    pd.device.random_matrix(nq, 1515, g.data_ptr(), 0)
    out = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    scratch = device_scratch(pd, nq, path="wht")
    pd.device.decompose(nq, g.data_ptr(), out.data_ptr(), scratch.data_ptr(), "gray", 0)
    ns = torch.from_numpy(np.sort(np.random.default_rng(15).choice(4**nq, 65536, replace=False))
                          .astype(np.int64)).to(cuda)
    walk = torch.empty(65536, dtype=torch.complex128, device=cuda)
    pd.device.coeff_batch(nq, g.data_ptr(), ns.data_ptr(), 65536, False, walk.data_ptr(), 0)
    torch.cuda.synchronize()
    assert same_values(out[ns].cpu().numpy(), walk.cpu().numpy())
    fro = float(torch.sum(torch.abs(g) ** 2))
    par = float(2**nq * torch.sum(torch.abs(out) ** 2))
    assert abs(fro - par) <= 1e-10 * fro
    del walk
    out2 = torch.empty_like(out)
    pd.device.decompose(nq, g.data_ptr(), out2.data_ptr(), scratch.data_ptr(), "wht", 0)
    torch.cuda.synchronize()
    err = float(torch.max(torch.abs(out2 - out)) / torch.max(torch.abs(out)))
    assert err <= TOL


def test_empty_and_single_string_batches(pd, cuda, port):
    rng = np.random.default_rng(3)
    g = normal_matrix(rng, 4)
    assert pd.coefficients(g, np.zeros(0, dtype=np.uint64)).shape == (0,)
    want = port.decompose(g)
    for n in (0, 1, 4**4 - 1):
        assert same_values(pd.coefficients(g, np.array([n], dtype=np.uint64)), want[[n]])


@pytest.mark.parametrize("nq,kind", [(5, "uniform"), (8, "one_xmask"), (9, "skewed"), (13, "uniform")])
def test_grouped_strings_equal_reference_order_walk(pd, cuda, nq, kind):
    """K3b (strings bucketed by X-mask, one CTA per bucket) must equal K3 (one thread per string
    straight from G, selected here with slow=True) bit for bit, for bucket shapes the bucketing
    can get wrong: a single X-mask holding every string, heavily skewed buckets, empty buckets,
    duplicates, and the size limits N=5 and N=13."""
    import torch
    rng = np.random.default_rng(nq)
    count = max(3 * 2**nq, 4096)
    if kind == "uniform":
        ns = rng.integers(0, 4**nq, count)
    elif kind == "one_xmask":   # X-mask 0b1011 only: digits X/Y at bits 0,1,3, I/Z elsewhere
        x = 0b1011
        z = rng.integers(0, 2**nq, count)
        ns = np.array([_n(x, int(zz), nq) for zz in z])
    else:                       # 90 % of the strings in 4 X-masks
        hot = rng.integers(0, 4**nq, 4)
        ns = np.where(rng.random(count) < 0.9, hot[rng.integers(0, 4, count)], rng.integers(0, 4**nq, count))
    ns = torch.from_numpy(ns.astype(np.int64)).to(cuda)
    g = torch.from_numpy(normal_matrix(rng, nq)).to(cuda)
    fast = torch.empty(count, dtype=torch.complex128, device=cuda)
    ref = torch.empty_like(fast)
    pd.device.coeff_batch(nq, g.data_ptr(), ns.data_ptr(), count, False, fast.data_ptr(), 0)
    pd.device.coeff_batch(nq, g.data_ptr(), ns.data_ptr(), count, True, ref.data_ptr(), 0)
    torch.cuda.synchronize()
    assert same_values(fast.cpu().numpy(), ref.cpu().numpy())


def _n(x, z, nq):
    """tensor number of X-mask x and Z-mask z: digit t = 2 z_t + (x_t ^ z_t)"""
    return sum((2 * ((z >> t) & 1) + (((x ^ z) >> t) & 1)) << (2 * t) for t in range(nq))


def test_blocked_scratch_matches_one_shot(pd, cuda):
    import torch
    nq = 11
    g = torch.from_numpy(normal_matrix(np.random.default_rng(11), nq)).to(cuda)
    full = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    scratch = device_scratch(pd, nq, path="wht")
    for path in ("gray", "wht"):
        pd.device.decompose(nq, g.data_ptr(), full.data_ptr(), scratch.data_ptr(), path, 0)
        for blocks in (2, 8, 64):
            out = torch.zeros_like(full)
            pd.device.decompose_blocked(nq, g.data_ptr(), out.data_ptr(), scratch.data_ptr(),
                                        16 * 4**nq // blocks, path, 0)
            torch.cuda.synchronize()
            assert torch.equal(out, full), (path, blocks)
    with pytest.raises(ValueError):
        pd.device.decompose_blocked(nq, g.data_ptr(), full.data_ptr(), scratch.data_ptr(),
                                    16 * 2**nq * 8, "gray", 0)


def test_n16_on_one_gpu_with_blocked_scratch(pd, cuda):
    """N=16, 4,294,967,296 coefficients: G and the coefficients take 64 GiB each, so the
    diagonals are processed in blocks of 4096 X-masks (16 GiB of scratch). Gray path checked
    against the reference-order walk (K3) on 2,048 seeded strings bit for bit, Parseval over the
    whole array, then the WHT path into the same buffer against the same sample and norm."""
    import torch
    nq = 16
    torch.cuda.empty_cache()  # earlier tests' cached blocks
    free, _ = torch.cuda.mem_get_info()
    if free < 150 * 2**30:
        pytest.skip("needs ~145 GiB of free device memory")
    g = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=cuda)
    pd.device.random_matrix(nq, 1616, g.data_ptr(), 0)
    out = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    scratch = device_scratch(pd, nq, 4096)
    pd.device.decompose_blocked(nq, g.data_ptr(), out.data_ptr(), scratch.data_ptr(),
                                scratch.numel() * 16, "gray", 0)
    ns = torch.from_numpy(np.sort(np.random.default_rng(16).choice(4**nq, 2048, replace=False))
                          .astype(np.int64)).to(cuda)
    walk = torch.empty(2048, dtype=torch.complex128, device=cuda)
    pd.device.coeff_batch(nq, g.data_ptr(), ns.data_ptr(), 2048, True, walk.data_ptr(), 0)
    torch.cuda.synchronize()
    gray_sample = out[ns].clone()
    assert same_values(gray_sample.cpu().numpy(), walk.cpu().numpy())
    fro = _sq_norm(g)
    par = 2**nq * _sq_norm(out)
    assert abs(fro - par) <= 1e-10 * fro
    pd.device.decompose_blocked(nq, g.data_ptr(), out.data_ptr(), scratch.data_ptr(),
                                scratch.numel() * 16, "wht", 0)
    torch.cuda.synchronize()
    err = float(torch.max(torch.abs(out[ns] - gray_sample)) / torch.max(torch.abs(gray_sample)))
    assert err <= TOL
    par2 = 2**nq * _sq_norm(out)
    assert abs(fro - par2) <= 1e-10 * fro


def _sq_norm(t):
    """sum |t|^2 in 2^26-element slices (no full-size temporary)"""
    v = t.reshape(-1)
    step = 1 << 26
    return float(sum(float(torch_sum_sq(v[i:i + step])) for i in range(0, v.numel(), step)))


def torch_sum_sq(v):
    import torch
    r = torch.view_as_real(v)
    return torch.sum(r * r)


def test_array_like_inputs_are_coerced_like_the_reference_binding(pd, cuda, port):
    """module.cpp:21 of the reference takes any array-like through pybind's forcecast to a
    C-contiguous complex128 array: lists, real or integer arrays, transposed / Fortran-ordered
    and strided views must all decompose exactly like their complex128 C-contiguous copy."""
    rng = np.random.default_rng(21)
    g = normal_matrix(rng, 4)
    want = port.decompose(np.ascontiguousarray(g))
    assert same_values(pd.decompose(g.tolist()), want)
    gt = np.ascontiguousarray(g.T)
    assert same_values(pd.decompose(g.T.T), want)
    assert same_values(pd.decompose(np.asfortranarray(g)), want)
    assert same_values(pd.decompose(gt.T), want)                      # non-contiguous view
    big = np.zeros((32, 32), dtype=complex)
    big[::2, ::2] = g
    assert same_values(pd.decompose(big[::2, ::2]), want)             # strided view
    r = rng.standard_normal((16, 16))
    assert same_values(pd.decompose(r), port.decompose(r.astype(complex)))
    i = rng.integers(-3, 4, (8, 8))
    assert same_values(pd.decompose(i), port.decompose(i.astype(complex)))
    assert same_values(pd.coefficients(g.tolist(), [0, 5, 255]), want[[0, 5, 255]])


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0, 0], [0] * 8])
@pytest.mark.parametrize("nq,path", [(9, "gray"), (12, "gray"), (12, "wht"), (13, "gray")])
def test_multi_device_context_matches_one_device(pd, cuda, devices, nq, path):
    """pd_ctx_create_multi on a list that repeats device 0: every virtual device gets its own
    streams and buffers (left uninitialised), uploads only the tiles (t ^ g, t) of G its
    X-masks touch and downloads its runs to their offsets — a missing tile or a misplaced run
    shows up as a mismatch. No kernel waits on another, so sharing one GPU is safe."""
    g = normal_matrix(np.random.default_rng(nq), nq)
    want = pd.decompose(g, path=path)
    got = pd.decompose(g, path=path, devices=devices)
    assert np.array_equal(got, want)


def test_random_sizes_paths_and_batches(pd, cuda, port):
    """Hypothesis-drawn sizes, paths, matrices and string batches against the oracle: Gray and
    naive paths and every batched string bit for bit, the WHT path within the tolerance."""
    from hypothesis import HealthCheck, given, settings
    from hypothesis import strategies as st

    @settings(max_examples=30, deadline=None, suppress_health_check=list(HealthCheck))
    @given(st.integers(1, 11), st.sampled_from(["gray", "wht", "naive"]), st.integers(0, 2**32 - 1),
           st.integers(0, 5000))
    def check(nq, path, seed, count):
        rng = np.random.default_rng(seed)
        g = rng.standard_normal((2**nq, 2**nq)) + 1j * rng.standard_normal((2**nq, 2**nq))
        if rng.random() < 0.3:  # small integers: every path is exact
            g = rng.integers(-4, 5, (2**nq, 2**nq)) + 1j * rng.integers(-4, 5, (2**nq, 2**nq))
        want = port.decompose(g)
        got = pd.decompose(g, path=path)
        if path == "wht":
            assert np.max(np.abs(got - want)) <= 1e-11 * max(np.max(np.abs(want)), 1e-300)
        else:
            assert same_values(got, want)
        ns = rng.integers(0, 4**nq, count).astype(np.uint64)
        assert same_values(pd.coefficients(g, ns), want[ns.astype(np.int64)])

    check()


def test_concurrent_callers(pd, cuda, port):
    """Host threads decomposing at once (one context per device, serialised by the C++ layer;
    the shared WHT stream pipeline and lazily set kernel attributes must not race)."""
    import threading
    rng = np.random.default_rng(77)
    mats = [normal_matrix(rng, nq) for nq in (6, 9, 10, 11)]
    want = [port.decompose(g) for g in mats]
    errors = []

    def work(k):
        try:
            for rep in range(3):
                g = mats[(k + rep) % len(mats)]
                w = want[(k + rep) % len(mats)]
                path = ("gray", "wht", "naive")[(k + rep) % 3]
                got = pd.decompose(g, path=path)
                ok = (np.max(np.abs(got - w)) <= 1e-11 * np.max(np.abs(w))) if path == "wht" \
                    else same_values(got, w)
                if not ok:
                    errors.append((k, rep, path))
        except Exception as exc:  # pragma: no cover - reported below
            errors.append((k, repr(exc)))

    threads = [threading.Thread(target=work, args=(k,)) for k in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("nq,count,n_x", [(8, 50, 3), (12, 200, 7), (14, 64, 64)])
def test_sparse_batches_use_gathered_diagonals(pd, cuda, port, nq, count, n_x):
    """Batches whose strings share few X-masks upload only those diagonals (pd_coeff_batch);
    every value must still equal the oracle bit for bit, duplicates and all."""
    rng = np.random.default_rng(count)
    g = port.random_matrix(nq, 99 + nq) if nq == 14 else normal_matrix(rng, nq)
    xs = rng.choice(2**nq, n_x, replace=False)
    zs = rng.integers(0, 2**nq, count)
    ns = np.array([_n(int(xs[k % n_x]), int(zs[k]), nq) for k in range(count)], dtype=np.uint64)
    got = pd.coefficients(g, ns)
    want = port.coeff_batch(g, ns)
    assert same_values(got, want)


@pytest.mark.parametrize("nq", [11, 12, 13])
def test_recompose_inverse_passes_round_trip(pd, cuda, port, nq):
    """N >= 11 recomposes through the chunked inverse WHT passes: G -> c -> G within 1e-12 of
    the largest element, and equal to the oracle's recompose on the same coefficients to the
    same tolerance (both sum in different orders)."""
    import torch
    rng = np.random.default_rng(nq)
    g = normal_matrix(rng, nq)
    c = port.decompose(g) if nq == 11 else pd.decompose(g)  # the GPU path is pinned elsewhere
    back = pd.recompose(c)
    scale = np.max(np.abs(g))
    assert np.max(np.abs(back - g)) <= 1e-12 * scale
    if nq == 11:
        assert np.max(np.abs(back - port.recompose(c))) <= 1e-12 * scale
    # device form with the documented scratch size
    cd = torch.from_numpy(c).to(cuda)
    gd = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=cuda)
    scr = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    pd.device.recompose(nq, cd.data_ptr(), gd.data_ptr(), scr.data_ptr(), 0)
    torch.cuda.synchronize()
    assert np.max(np.abs(gd.cpu().numpy() - g)) <= 1e-12 * scale


def test_random_matrix_api_matches_reference_generator(pd, cuda, port):
    for nq, seed in ((1, 3), (5, 77), (9, pd.matrix_seed(20260823, 9, 0))):
        assert np.array_equal(pd.random_matrix(nq, seed).view(np.uint64),
                              port.random_matrix(nq, seed).view(np.uint64))


def test_host_path_falls_back_to_blocked_scratch_when_memory_is_short(cuda):
    """With G and the coefficients resident but no room for every diagonal (N=16 on one B200),
    pd_decompose uploads, decomposes in X-mask blocks sized to the free memory and downloads.
    Simulated at N=14 in a fresh process by filling all but ~10 GiB of the device first; the
    result must equal the normal pipelined path bit for bit."""
    import subprocess
    import sys
    import torch
    torch.cuda.empty_cache()  # this process's cached blocks (the N=16 test leaves ~144 GiB)
    if torch.cuda.mem_get_info()[0] < 40 * 2**30:
        pytest.skip("needs ~40 GiB of free device memory")
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2401_16378_b200 as pd
nq = 14
g = pd.random_matrix(nq, 4141)
free, _ = torch.cuda.mem_get_info()
filler = torch.empty(free - (10 << 30), dtype=torch.uint8, device="cuda")
a = pd.decompose(g)
del filler
torch.cuda.empty_cache()
b = pd.decompose(g)
assert np.array_equal(a, b)
print("ok")
''' % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


def test_k2s_c_shards_run_bits_n14(pd, cuda):
    """The kernel configuration every rank of a 2/4/8-GPU run executes at N=14: K2s-c (each
    rank's 8192 / 4096 / 2048 X-masks exceed gray_share_c_min_xmasks(14)) with run_bits 1..3,
    in both output layouts (rank 0 writes GLOBAL in place, the others pack RUNS). Emulated shard
    by shard on one GPU and compared bit for bit with the one-shot decomposition."""
    import torch
    nq = 14
    g = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=cuda)
    pd.device.random_matrix(nq, pd.matrix_seed(20260823, nq, 0), g.data_ptr(), 0)
    full = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    scratch = device_scratch(pd, nq)
    pd.device.decompose(nq, g.data_ptr(), full.data_ptr(), scratch.data_ptr(), "gray", 0)
    out = torch.empty_like(full)
    for p in (1, 2, 3):
        xc = 2 ** (nq - p)
        rl = 4 ** (nq - p)
        packed = torch.empty(4**nq >> p, dtype=torch.complex128, device=cuda)
        out.zero_()
        for shard in range(2**p):
            pd.device.diag_gather(nq, g.data_ptr(), shard * xc, xc, scratch.data_ptr(), 0)
            if shard == 0:   # rank 0: GLOBAL, in place
                pd.device.xmask_coeffs(nq, scratch.data_ptr(), 0, xc, p, out.data_ptr(), "global",
                                       "gray", 0)
            else:            # the other ranks: RUNS, packed for the gather
                pd.device.xmask_coeffs(nq, scratch.data_ptr(), shard * xc, xc, p, packed.data_ptr(),
                                       "runs", "gray", 0)
                for r in range(2**p):
                    o = pd.device.run_offset(nq, p, shard, r)
                    out[o:o + rl] = packed[r * rl:(r + 1) * rl]
        torch.cuda.synchronize()
        assert torch.equal(out, full), p
        # and every shard in the other layout too
        out.zero_()
        for shard in range(2**p):
            pd.device.diag_gather(nq, g.data_ptr(), shard * xc, xc, scratch.data_ptr(), 0)
            if shard == 0:
                pd.device.xmask_coeffs(nq, scratch.data_ptr(), 0, xc, p, packed.data_ptr(), "runs",
                                       "gray", 0)
                for r in range(2**p):
                    o = pd.device.run_offset(nq, p, 0, r)
                    out[o:o + rl] = packed[r * rl:(r + 1) * rl]
            else:
                pd.device.xmask_coeffs(nq, scratch.data_ptr(), shard * xc, xc, p, out.data_ptr(),
                                       "global", "gray", 0)
        torch.cuda.synchronize()
        assert torch.equal(out, full), p
        del packed


def test_k2s_c_segment_host_pipeline_n15(pd, cuda):
    """N=15 through the host API: the pipeline's final-segment launches (1024 X-masks per
    download block >= gray_share_c_min_xmasks(15)) run the K2s-c segment instantiation
    (pd_k2cseg.cu); the result must equal the device-resident one-shot decomposition."""
    import torch
    nq = 15
    torch.cuda.empty_cache()
    if torch.cuda.mem_get_info()[0] < 120 * 2**30:
        pytest.skip("needs ~112 GiB of free device memory")
    g = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=cuda)
    pd.device.random_matrix(nq, 1515, g.data_ptr(), 0)
    out = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    scratch = device_scratch(pd, nq)
    pd.device.decompose(nq, g.data_ptr(), out.data_ptr(), scratch.data_ptr(), "gray", 0)
    torch.cuda.synchronize()
    del scratch
    gh = g.cpu().numpy()
    del g
    torch.cuda.empty_cache()
    host = pd.decompose(gh)
    del gh
    want = out.cpu().numpy()
    assert np.array_equal(host.view(np.uint64), want.view(np.uint64))


def test_full_n12_config4_full_array(pd, cuda, port):
    """BASELINE configs[3]: every one of the 16,777,216 coefficients of an N=12 N(0,1) matrix
    equal to the oracle (IEEE ==), through the host API and the serial driver alias"""
    g = normal_matrix(np.random.default_rng(412), 12)
    want = port.decompose(g)
    assert same_values(pd.decompose(g), want)
    assert same_values(pd.decompose(g, serial=True, threads=0), want)


@pytest.mark.parametrize("nq", range(1, 7))
def test_serial_quaternary_driver(pd, cuda, golden, nq):
    """decompose(g, serial=True) (module.cpp:56-60 -> decompose_serial_quaternary,
    decompose.cpp:133-152) gives the reference's serial output; it ignores `threads`, and the
    parallel driver rejects threads=0 (decompose.cpp:98-99)"""
    g = golden[f"normal{nq}_matrix"]
    assert same_values(pd.decompose(g, serial=True), golden[f"normal{nq}_serial"])
    assert same_values(pd.decompose(g, threads=0, serial=True), golden[f"normal{nq}_serial"])
    with pytest.raises(ValueError):
        pd.decompose(g, threads=0)


def test_random_large_sizes_host_buffers(pd, cuda, port):
    """Hypothesis-drawn N = 12 … 14 through the public API, with the matrix and the result in
    pageable or page-locked host memory (pinned slot rings vs direct DMA), matrix kinds that
    stress the sums (N(0,1), small integers: exact partial sums, real, Hermitian), Gray or WHT:
    4096 seeded coefficients against the oracle (Gray bit for bit, WHT within 1e-11·max|c|)
    plus Parseval over the whole array."""
    import torch
    from hypothesis import HealthCheck, given, settings
    from hypothesis import strategies as st

    @settings(max_examples=8, deadline=None, suppress_health_check=list(HealthCheck))
    @given(st.sampled_from([12, 12, 13, 13, 14]), st.sampled_from(["gray", "gray", "wht"]),
           st.sampled_from(["normal", "integer", "real", "hermitian"]), st.booleans(), st.booleans(),
           st.integers(0, 2**32 - 1))
    def check(nq, path, kind, pin_in, pin_out, seed):
        rng = np.random.default_rng(seed)
        d = 2**nq
        g = torch.empty((d, d), dtype=torch.complex128, pin_memory=pin_in).numpy()
        if kind == "integer":
            g.real = rng.integers(-4, 5, (d, d))
            g.imag = rng.integers(-4, 5, (d, d))
        else:
            g.real = rng.standard_normal((d, d))
            g.imag = 0.0 if kind == "real" else rng.standard_normal((d, d))
            if kind == "hermitian":
                g[...] = (g + g.conj().T) / 2
        out = torch.empty(4**nq, dtype=torch.complex128, pin_memory=True).numpy() if pin_out else \
            np.empty(4**nq, dtype=np.complex128)
        out[...] = np.nan
        pd.decompose(g, path=path, out=out)
        ns = np.sort(rng.choice(4**nq, 4096, replace=False)).astype(np.uint64)
        want = port.coeff_batch(g, ns)
        got = out[ns.astype(np.int64)]
        if path == "gray":
            assert same_values(got, want)
        else:
            assert np.max(np.abs(got - want)) <= 1e-11 * max(np.max(np.abs(want)), 1e-300)
        fro = float(np.vdot(g.ravel(), g.ravel()).real)
        par = float(d * np.vdot(out, out).real)
        assert abs(fro - par) <= 1e-10 * fro

    check()
