"""The drop-in boundary, checked without a GPU: the C ABI exports, the Python surface of
proj/bindings/module.cpp:87-121, its error mapping, and the host-side index algebra."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle as O

HEADER = os.path.join(ROOT, "include", "pd_api.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^PD_EXPORT [\w\s\*]*?\b(pd_\w+)\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol(pd):
    syms = declared_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(pd.LIBRARY_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    lib.pd_api_version.restype = ctypes.c_int
    assert lib.pd_api_version() == 3
    lib.pd_last_error.restype = ctypes.c_char_p


def test_c_abi_validation_without_compute(pd):
    lib = ctypes.CDLL(pd.LIBRARY_PATH)
    lib.pd_last_error.restype = ctypes.c_char_p
    lib.pd_scratch_bytes.restype = ctypes.c_uint64
    lib.pd_scratch_bytes.argtypes = [ctypes.c_uint, ctypes.c_uint64, ctypes.c_int]
    assert lib.pd_scratch_bytes(14, 1 << 14, 0) == 16 * 4**14
    assert lib.pd_scratch_bytes(14, 1 << 14, 2) == 0
    # qubit-count contract of matrix.cpp:10-19, checked before any device work
    lib.pd_random_matrix_device.argtypes = [ctypes.c_uint, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    assert lib.pd_random_matrix_device(0, 1, None, None) == -1
    assert lib.pd_random_matrix_device(33, 1, None, None) == -1
    assert lib.pd_random_matrix_device(32, 1, None, None) == -2
    assert b"32 qubits" in lib.pd_last_error()


def test_python_surface_matches_reference_module(pd):
    # the names re-exported by proj/python/paulidecomp/__init__.py:7-33
    for name in ("FormatError", "__version__", "coefficient", "decompose", "flipped_bit_index",
                 "gray_code", "index_to_label", "label_to_index", "oracle_coefficient",
                 "recompose", "xy_mask"):
        assert hasattr(pd, name), name
    assert issubclass(pd.FormatError, ValueError)


def test_label_helpers_match_reference_golden(pd, golden):
    for lab, n in zip(golden["labels"], golden["label_index"]):
        assert pd.label_to_index(str(lab), len(str(lab))) == int(n)
        assert pd.index_to_label(int(n), len(str(lab))) == str(lab)
    for k, g, f in zip(golden["gray_k"], golden["gray_code"], golden["flipped_bit"]):
        assert pd.gray_code(int(k)) == int(g)
        assert pd.flipped_bit_index(int(k)) == int(f)
    for n, m in zip(golden["xy_mask_n"], golden["xy_mask_4"]):
        assert pd.xy_mask(int(n), 4) == int(m)
    # test_smoke.py:89-94
    assert pd.label_to_index("XY", 2) == 6 and pd.index_to_label(6, 2) == "XY"
    assert pd.gray_code(3) == 2 and pd.flipped_bit_index(3) == 2 and pd.xy_mask(6, 2) == 3


def test_errors_surface_as_python_exceptions(pd):
    # test_smoke.py:97-105 — raised by validation before any device work
    with pytest.raises(ValueError):
        pd.label_to_index("XQ", 2)
    with pytest.raises(pd.FormatError):
        pd.label_to_index("XYZ", 2)
    with pytest.raises(ValueError):
        pd.decompose(np.zeros((3, 3), dtype=complex))
    with pytest.raises(ValueError):
        pd.decompose(np.zeros((2, 4), dtype=complex))
    with pytest.raises(ValueError):
        pd.decompose(np.zeros((1, 1), dtype=complex))
    with pytest.raises(ValueError):
        pd.recompose(np.zeros(7, dtype=complex))
    with pytest.raises(ValueError):
        pd.recompose(np.zeros(8, dtype=complex))
    with pytest.raises(ValueError):
        pd.decompose(np.eye(4, dtype=complex), threads=0)
    with pytest.raises(ValueError):
        pd.decompose(np.eye(4, dtype=complex), path="fft")
    with pytest.raises(ValueError):
        pd.index_to_label(16, 2)


def test_no_cpu_fallback_without_gpu(pd):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CPU path"):
        pd.decompose(np.eye(4, dtype=complex))
    with pytest.raises(RuntimeError):
        pd.coefficient(np.eye(2, dtype=complex), 0)


def test_run_offsets_partition_the_coefficient_array(pd):
    # shard g of P = 2^p owns the 2^p runs of 4^(N-p) coefficients whose top digits
    # are 2 z_t + (x_t ^ z_t) with x's top bits = g
    for nq in (3, 4, 6):
        for p in range(0, 4):
            if p > nq:
                continue
            run = 4 ** (nq - p)
            seen = []
            for g in range(1 << p):
                for r in range(1 << p):
                    off = pd.device.run_offset(nq, p, g, r)
                    assert off % run == 0
                    seen.append(off)
                    # every n of the run has its X-mask in shard g and Z-mask top bits r
                    ns = np.arange(off, off + run, dtype=np.uint64)
                    for n in ns[:: max(1, run // 7)]:
                        x = O.port().xy_mask(int(n), nq)
                        z = sum((((int(n) >> (2 * t + 1)) & 1) << t) for t in range(nq))
                        assert x >> (nq - p) == g and z >> (nq - p) == r
            assert sorted(seen) == list(range(0, 4**nq, run))


def test_product_package_never_touches_the_oracle():
    pkg = os.path.join(ROOT, "paper_2401_16378_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".h", ".hpp")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "libpd_oracle" not in text and "libpdref" not in text, f


def test_matrix_seed_matches_reference(pd, port):
    # bench.cpp:42-46, used by bench.py for the BASELINE configs[4] matrix
    for seed, nq, rep in [(20260823, 14, 0), (1, 1, 0), (1, 5, 19), (2**63 + 5, 12, 7)]:
        assert pd.matrix_seed(seed, nq, rep) == port.matrix_seed(seed, nq, rep)


def test_bench_does_not_use_the_oracle_outside_its_cpu_legs():
    src = open(os.path.join(ROOT, "bench.py")).read()
    run_ours = src[src.index("def run_ours("):src.index("def side_configs(")]
    assert "oracle" not in run_ours


def test_c_abi_rejects_null_buffers_before_device_work(pd):
    lib = ctypes.CDLL(pd.LIBRARY_PATH)
    lib.pd_last_error.restype = ctypes.c_char_p
    vp = ctypes.c_void_p
    lib.pd_coeff_batch.argtypes = [vp, ctypes.c_uint, vp, vp, ctypes.c_uint64, vp]
    assert lib.pd_coeff_batch(None, 4, None, None, 3, None) == -1
    lib.pd_coeff_batch_device.argtypes = [ctypes.c_uint, vp, vp, ctypes.c_uint64, ctypes.c_int, vp, vp]
    assert lib.pd_coeff_batch_device(4, None, None, 3, 0, None, None) == -1
    lib.pd_decompose_device.argtypes = [ctypes.c_uint, vp, vp, vp, ctypes.c_int, vp]
    assert lib.pd_decompose_device(4, None, None, None, 0, None) == -1
    lib.pd_coeff.argtypes = [vp, ctypes.c_uint, vp, ctypes.c_uint64, ctypes.c_int, vp]
    assert lib.pd_coeff(None, 4, None, 0, 0, None) == -1
    assert b"null" in lib.pd_last_error()
    lib.pd_ctx_create_multi.argtypes = [vp, ctypes.c_int, vp]
    out = vp()
    devs = (ctypes.c_int * 3)(0, 0, 0)
    assert lib.pd_ctx_create_multi(devs, 3, ctypes.byref(out)) == -1   # not a power of two
