"""File formats (proj/docs/formats.md) against the reference's own readers and writers
(proj/src/io.cpp via oracle/_ref), byte for byte, plus the GPU file path (decompose_file,
the pdb200 CLI). CPU tests need only the host code; `gpu` tests decompose on the device."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, normal_matrix

CLI = os.path.join(ROOT, "paper_2401_16378_b200", "pdb200")


def special_matrix(nq, seed):
    g = normal_matrix(np.random.default_rng(seed), nq)
    flat = g.reshape(-1)
    flat[0] = complex(-0.0, 0.0)
    if flat.size > 3:
        flat[1] = complex(5e-324, -0.0)       # subnormal, negative zero
        flat[2] = complex(1e300, -2.5e-8)
        flat[3] = complex(3.0, -7.0)          # integral values get ".0"
    return g


def test_format_double_matches_reference(pd, ref):
    rng = np.random.default_rng(0)
    vals = [0.0, -0.0, 1.0, -2.0, 0.1, 1e-320, 5e-324, 1.7976931348623157e308, 123456789.0,
            1e16, 1e22, 2.5e-8, float(2**53), -1.5]
    vals += list(rng.standard_normal(200)) + list(rng.standard_normal(50) * 1e-200)
    for v in vals:
        assert pd.format_double(v) == ref.format_double(v), v


@pytest.mark.parametrize("binary", [False, True])
@pytest.mark.parametrize("nq", [1, 2, 4])
def test_matrix_files_byte_identical(pd, ref, tmp_path, binary, nq):
    g = special_matrix(nq, 40 + nq)
    ours, theirs = str(tmp_path / "ours"), str(tmp_path / "theirs")
    fmt = "binary" if binary else "text"
    pd.write_matrix(g, ours, fmt)
    ref.write_matrix(g, theirs, binary)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    back = pd.read_matrix(theirs, fmt)
    assert np.array_equal(back.view(np.uint64), g.view(np.uint64))
    assert np.array_equal(ref.read_matrix(ours, binary).view(np.uint64), g.view(np.uint64))


@pytest.mark.parametrize("threshold", [0.0, 0.05, 0.3])
def test_coefficient_csv_byte_identical(pd, ref, golden, tmp_path, threshold):
    for key in ("normal4_coeffs", "unif5_coeffs", "kat_coeffs"):
        c = golden[key]
        ours, theirs = str(tmp_path / "o.csv"), str(tmp_path / "t.csv")
        n1 = pd.write_coefficients(c, ours, threshold)
        n2 = ref.write_coefficients(c, theirs, threshold)
        assert n1 == n2
        assert open(ours, "rb").read() == open(theirs, "rb").read(), key
        back = pd.read_coefficients(theirs)
        kept = np.abs(c) > threshold if threshold > 0 else np.ones(c.size, bool)
        assert np.array_equal(back[kept], c[kept]) and np.all(back[~kept] == 0)
        assert np.array_equal(ref.read_coefficients(ours), back)


def test_text_reader_variants_and_errors(pd, tmp_path):
    p = str(tmp_path / "m.txt")
    # headerless square layout, CRLF, blank lines, leading '+', exponent signs
    open(p, "w").write("+1.0+0.0j 2e-1-3e+2j\r\n\r\n-0.5+0.25j 4.0-0.0j\r\n")
    g = pd.read_matrix(p, "text")
    assert g.shape == (2, 2) and g[0, 1] == complex(0.2, -300.0) and g[1, 0] == complex(-0.5, 0.25)
    bad = {
        "3x3": "1+0j 1+0j 1+0j\n1+0j 1+0j 1+0j\n1+0j 1+0j 1+0j\n",
        "short row": "PAULIDECOMP-MAT v1 N=1\n1.0+0.0j\n2.0+0.0j 3.0+0.0j\n",
        "extra row": "PAULIDECOMP-MAT v1 N=1\n1+0j 1+0j\n1+0j 1+0j\n1+0j 1+0j\n",
        "bad header": "PAULIDECOMP-MAT v2 N=1\n1+0j 1+0j\n1+0j 1+0j\n",
        "non-finite": "PAULIDECOMP-MAT v1 N=1\ninf+0j 1+0j\n1+0j 1+0j\n",
        "bad token": "PAULIDECOMP-MAT v1 N=1\n1.0 1+0j\n1+0j 1+0j\n",
        "empty": "",
    }
    for why, text in bad.items():
        open(p, "w").write(text)
        with pytest.raises(ValueError):
            pd.read_matrix(p, "text")


def test_binary_reader_errors(pd, tmp_path):
    p = str(tmp_path / "m.bin")
    good = b"PDMAT-V1" + (1).to_bytes(8, "little") + np.arange(8, dtype=np.float64).tobytes()
    open(p, "wb").write(good)
    assert pd.read_matrix(p, "binary")[1, 1] == complex(6, 7)
    for why, blob in {"magic": b"PDMAT-V2" + good[8:], "truncated": good[:-8],
                      "trailing": good + b"\0", "N=0": b"PDMAT-V1" + bytes(8) + good[16:],
                      "nan": good[:16] + np.array([np.nan] + [0.0] * 7).tobytes()}.items():
        open(p, "wb").write(blob)
        with pytest.raises(ValueError):
            pd.read_matrix(p, "binary")


def test_coefficient_reader_errors(pd, tmp_path):
    p = str(tmp_path / "c.csv")
    open(p, "w").write("pauli,re,im\nXY,1.0,0.0\nZZ,0.5,-0.5\n")  # header line optional
    c = pd.read_coefficients(p)
    assert c.size == 16 and c[6] == 1.0 and c[15] == complex(0.5, -0.5)
    for text in ("pauli,re,im\nXY,1.0\n", "pauli,re,im\nXY,1,0\nXY,2,0\n", "pauli,re,im\nXY,1,0\nX,1,0\n",
                 "# PAULIDECOMP-COEF v1 N=2\npauli,re,im\nXQ,1,0\n", "pauli,re,im\n",
                 "# PAULIDECOMP-COEF v1 N=2\npauli,re,im\nXY,nan,0\n", "re,im\n"):
        open(p, "w").write(text)
        with pytest.raises(ValueError):
            pd.read_coefficients(p)


# ---------------- GPU file path ----------------

@pytest.mark.gpu
@pytest.mark.parametrize("threshold", [0.0, 0.02])
@pytest.mark.parametrize("fmt", ["binary", "text"])
def test_decompose_file_matches_reference_cli_output(pd, ref, cuda, tmp_path, threshold, fmt):
    # the reference CLI's decompose = read_matrix -> decompose_parallel -> write_coefficients
    g = normal_matrix(np.random.default_rng(77), 7)
    src = str(tmp_path / f"g.{fmt}")
    pd.write_matrix(g, src, fmt)
    ours, theirs = str(tmp_path / "o.csv"), str(tmp_path / "t.csv")
    n = pd.decompose_file(src, ours, fmt, threshold)
    ref.write_coefficients(ref.decompose(ref.read_matrix(src, fmt == "binary")), theirs, threshold)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert n == len(open(ours).read().splitlines()) - 2


@pytest.mark.gpu
def test_decompose_file_threshold_selection_large(pd, cuda, port, tmp_path):
    # N=11: 4.2M coefficients selected on the GPU; the kept set must equal |c| > eps exactly
    g = normal_matrix(np.random.default_rng(11), 11)
    src, out = str(tmp_path / "g.bin"), str(tmp_path / "c.csv")
    pd.write_matrix(g, src, "binary")
    eps = 0.01
    n = pd.decompose_file(src, out, "binary", eps)
    c = pd.decompose(g)
    assert n == int(np.sum(np.abs(c) > eps))
    back = pd.read_coefficients(out)
    keep = np.abs(c) > eps
    assert np.array_equal(back[keep], c[keep]) and np.all(back[~keep] == 0)


@pytest.mark.gpu
def test_decompose_file_rejects_non_finite_on_device(pd, cuda, tmp_path):
    g = normal_matrix(np.random.default_rng(5), 6)
    g[17, 3] = complex(np.inf, 0)
    src = str(tmp_path / "bad.bin")
    with open(src, "wb") as f:  # written raw: the writer itself does not validate
        f.write(b"PDMAT-V1" + (6).to_bytes(8, "little") + g.tobytes())
    with pytest.raises(ValueError, match="row 17, column 3"):
        pd.decompose_file(src, str(tmp_path / "c.csv"), "binary", 0.0)


@pytest.mark.gpu
def test_cli_subcommands(pd, ref, cuda, tmp_path):
    g = normal_matrix(np.random.default_rng(3), 5)
    src, csv, back = str(tmp_path / "g.bin"), str(tmp_path / "c.csv"), str(tmp_path / "b.txt")
    pd.write_matrix(g, src, "binary")
    r = subprocess.run([CLI, "decompose", "--in", src, "--format", "binary", "--out", csv],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stderr.startswith("N=5 nonzero=1024 seconds=")
    theirs = str(tmp_path / "t.csv")
    ref.write_coefficients(ref.decompose(g), theirs)
    assert open(csv, "rb").read() == open(theirs, "rb").read()
    r = subprocess.run([CLI, "recompose", "--in", csv, "--out", back], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stderr
    np.testing.assert_allclose(pd.read_matrix(back, "text"), g, rtol=0, atol=1e-12)
    r = subprocess.run([CLI, "coeff", "XYZIX", "--in", src, "--format", "binary"], capture_output=True,
                       text=True, timeout=120)
    want = ref.coeff_fast(g, pd.label_to_index("XYZIX", 5))
    assert r.returncode == 0 and r.stdout.strip() == f"{ref.format_double(want.real)},{ref.format_double(want.imag)}"
    for args in (["decompose"], ["decompose", "--in", "/nonexistent"], ["frobnicate"],
                 ["decompose", "--in", src, "--eps", "-1"]):
        assert subprocess.run([CLI, *args], capture_output=True, timeout=60).returncode == 1, args


def _same_outcome(ours, theirs):
    """Both readers raise ValueError, or both return bit-identical arrays."""
    try:
        want = theirs()
    except ValueError:
        with pytest.raises(ValueError):
            ours()
        return
    got = ours()
    assert got.shape == want.shape and np.array_equal(got.view(np.uint64), want.view(np.uint64))


MATRIX_TEXTS = [
    "PAULIDECOMP-MAT v1 N=1\n1+2j 3-4j\n5e-1+6E+2j -0-0j\n",
    "PAULIDECOMP-MAT v1 N=1   \n\n1+2j\t3-4j  \n\n5+6j -7-8j\n\n\n",
    "\nPAULIDECOMP-MAT v1 N=1\n1+2j 3-4j\n5+6j 7+8j\n",        # header not on the first line
    "PAULIDECOMP-MAT v1 N=1\n1+2j 3-4j 9+9j\n5+6j 7+8j\n",     # surplus entry
    "PAULIDECOMP-MAT v1 N=0\n",
    "PAULIDECOMP-MAT v1 N=33\n",
    "PAULIDECOMP-MAT v1 N=1x\n1+2j 3-4j\n5+6j 7+8j\n",
    "PAULIDECOMP-MAT v1 N=2\n1+2j 3-4j\n5+6j 7+8j\n",          # truncated
    "1+2j 3-4j\n5+6j 7+8j\n\n\n",                               # headerless 2x2
    "\n\n1+2j 3-4j\n\n5+6j 7+8j\n",
    "1+2j 3-4j\n5+6j\n",
    "1+2j\n",
    "+1.5e+3-2.5e-3j +0+0j\n-1-1j 1e308+1e-308j\n",
    "1+2 3-4j\n5+6j 7+8j\n",
    "1+2j 3--4j\n5+6j 7+8j\n",
    "1e+2j 3-4j\n5+6j 7+8j\n",
    "nan+0j 3-4j\n5+6j 7+8j\n",
    "1+infj 3-4j\n5+6j 7+8j\n",
    "0x1p3+0j 3-4j\n5+6j 7+8j\n",
    "   \n \t \n",
    "1+2j 3-4j\r\n5+6j 7+8j\r\n\r\n",
]

COEF_TEXTS = [
    "# PAULIDECOMP-COEF v1 N=2\npauli,re,im\nXY,1.0,0.0\nZI,-0.5,2e-3\n",
    "pauli,re,im\nXY,1.0,0.0\n\nZI,-0.5,2e-3\n\n",
    "pauli,re,im\nZI,1,0\nXY,2,0\n",                            # unsorted records are accepted
    "pauli,re,im\nXY,1,0\nXY,2,0\n",
    "pauli,re,im\nXY,1,0\nZI,1,0\nXY,3,0\n",
    "pauli,re,im\nXY,1,0,0\n",
    "pauli,re,im\nXY,1\n",
    "pauli,re,im\nXQ,1,0\n",
    "pauli,re,im\n,1,0\n",
    "# PAULIDECOMP-COEF v1 N=3\npauli,re,im\nXY,1,0\n",
    "# PAULIDECOMP-COEF v1 N=2\n\npauli,re,im\nXY,1,0\n",
    "# PAULIDECOMP-COEF v2 N=2\npauli,re,im\n",
    "# PAULIDECOMP-COEF v1 N=2\npauli,re,im\n",
    "pauli,re,im\r\nXY,+1.0,-0.0\r\n",
    "pauli,re,im\nXY,inf,0\n",
    "pauli,re,im\nXY, 1,0\n",
    "pauli, re,im\nXY,1,0\n",
    "",
]


@pytest.mark.parametrize("k", range(len(MATRIX_TEXTS)))
def test_text_matrix_reader_agrees_with_reference(pd, ref, tmp_path, k):
    p = str(tmp_path / "m.txt")
    open(p, "w", newline="").write(MATRIX_TEXTS[k])
    _same_outcome(lambda: pd.read_matrix(p, "text"), lambda: ref.read_matrix(p, False))


@pytest.mark.parametrize("k", range(len(COEF_TEXTS)))
def test_coefficient_reader_agrees_with_reference(pd, ref, tmp_path, k):
    p = str(tmp_path / "c.csv")
    open(p, "w", newline="").write(COEF_TEXTS[k])
    _same_outcome(lambda: pd.read_coefficients(p), lambda: ref.read_coefficients(p))


@pytest.mark.gpu
def test_cli_bench_csv_schema(pd, port, cuda, tmp_path):
    """`pdb200 bench`: docs/formats.md's benchmark CSV — per (N, path) one row per repetition
    (the matrix_seed of that repetition, an empty stddev field) and then the rep = -1 summary
    (master seed, mean, sample stddev); paths fast / slow / serial-quaternary with the exact
    multiplication counts of proj/README.md:115-120; only the timing fields vary between runs."""
    import csv as csvmod
    outs = []
    for k in range(2):
        out = str(tmp_path / f"b{k}.csv")
        r = subprocess.run([CLI, "bench", "--n-min", "1", "--n-max", "4", "--reps", "3", "--seed", "11",
                            "--out", out], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        outs.append(list(csvmod.reader(open(out))))
    a, b = outs
    assert a[0] == ["N", "path", "threads", "rep", "seed", "seconds", "mult_count", "seconds_stddev"]
    assert len(a) == 1 + 4 * 3 * 4 and len(b) == len(a)
    counts = {"fast": lambda n: 4**n * (n + 2 * 2**n - 1), "slow": lambda n: 4**n * (n + 1) * 2**n,
              "serial-quaternary": lambda n: n + 4**n * (2 * 2**n - 1) + (4**n - 1)}
    for ra, rb in zip(a[1:], b[1:]):
        assert [ra[k] for k in (0, 1, 2, 3, 4, 6)] == [rb[k] for k in (0, 1, 2, 3, 4, 6)]
        nq, path, rep, seed = int(ra[0]), ra[1], int(ra[3]), int(ra[4])
        assert int(ra[6]) == counts[path](nq) and float(ra[5]) > 0
        if rep >= 0:
            assert seed == port.matrix_seed(11, nq, rep) and ra[7] == ""
        else:
            assert seed == 11 and float(ra[7]) >= 0
    for args in (["bench", "--n-max", "9"], ["bench", "--reps", "0"], ["bench", "--n-min", "3", "--n-max", "2"],
                 ["bench", "--seed", "-1"]):
        assert subprocess.run([CLI, *args], capture_output=True, timeout=60).returncode == 1, args


@pytest.mark.parametrize("nq,cells", [(4, [(5, 2)]), (10, [(1000, 7), (300, 1023), (900, 0)])])
def test_binary_reader_reports_first_non_finite(pd, tmp_path, nq, cells):
    # the binary reader fills the array in place and scans it on several threads (N=10: 2^20
    # elements); the reported element is the first in row-major order, like the text reader's
    g = normal_matrix(np.random.default_rng(nq), nq)
    for r, c in cells:
        g[r, c] = complex(0.0, np.inf) if r % 2 else complex(np.nan, 0.0)
    p = str(tmp_path / "m.bin")
    with open(p, "wb") as f:
        f.write(b"PDMAT-V1" + nq.to_bytes(8, "little") + g.tobytes())
    r, c = min(cells)
    with pytest.raises(ValueError, match=f"row {r}, column {c}$"):
        pd.read_matrix(p, "binary")
    g2 = normal_matrix(np.random.default_rng(nq + 1), nq)
    with open(p, "wb") as f:
        f.write(b"PDMAT-V1" + nq.to_bytes(8, "little") + g2.tobytes())
    back = pd.read_matrix(p, "binary")
    assert back.shape == g2.shape and np.array_equal(back.view(np.uint64), g2.view(np.uint64))
