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


@pytest.mark.gpu
def test_cli_bench_csv(pd, port, cuda, tmp_path):
    """`pdb200 bench` follows the reference's harness (main.cpp:110-128, bench.cpp:60-150): same
    options, same generator seeds, same CSV schema, one mean row (rep -1) per (N, path) with
    the sample stddev; the device paths must agree (the harness throws otherwise)."""
    import csv as csvmod
    out = str(tmp_path / "bench.csv")
    r = subprocess.run([CLI, "bench", "--n-min", "1", "--n-max", "6", "--reps", "3", "--seed", "7",
                        "--out", out], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = list(csvmod.reader(open(out)))
    assert rows[0] == ["N", "path", "threads", "rep", "seed", "seconds", "mult_count", "seconds_stddev"]
    body = rows[1:]
    assert len(body) == 6 * 3 * 4
    for row in body:
        nq, path, rep, seed = int(row[0]), row[1], int(row[3]), int(row[4])
        assert path in ("gray", "wht", "naive")
        if rep >= 0:
            assert seed == port.matrix_seed(7, nq, rep) and row[7] == ""
        else:
            assert seed == 7 and float(row[7]) >= 0.0
        if path == "gray":
            assert int(row[6]) == 4**nq * (nq + 2 * 2**nq - 1)
    for args in (["bench", "--n-max", "15"], ["bench", "--reps", "0"], ["bench", "--n-min", "3", "--n-max", "2"]):
        assert subprocess.run([CLI, *args], capture_output=True, timeout=60).returncode == 1, args
