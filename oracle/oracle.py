"""ctypes front for the test-only checkers built by oracle/Makefile.

TEST INFRASTRUCTURE ONLY (see oracle/pd_oracle.c). Importable from tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.
The product package never imports this module.

Two libraries:
  * ``port()``      -> oracle/_build/libpd_oracle.so, the C restatement.
  * ``reference()`` -> oracle/_ref/libpdref.so, the reference's own proj/src
                       compiled unmodified (None when it was never built).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libpd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpdref.so")

_u64 = ctypes.c_uint64
_uint = ctypes.c_uint
_dp = ctypes.POINTER(ctypes.c_double)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def _ptr(a: np.ndarray, typ=_dp):
    return a.ctypes.data_as(typ)


def build(reference: bool | None = None) -> None:
    """Compile the C restatement (and the reference shim when its sources exist)."""
    targets = ["oracle"]
    if reference is None:
        reference = os.path.isdir("/root/reference/proj/src")
    if reference:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _as_c128(g) -> np.ndarray:
    g = np.ascontiguousarray(g, dtype=np.complex128)
    return g


class Port:
    """The C restatement (oracle/pd_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(reference=False)
        lib = ctypes.CDLL(path)
        lib.pdo_xy_mask.restype = _u64
        lib.pdo_xy_mask.argtypes = [_u64, _uint]
        lib.pdo_initial_phase.restype = _uint
        lib.pdo_initial_phase.argtypes = [_u64, _uint]
        lib.pdo_gray_code.restype = _u64
        lib.pdo_gray_code.argtypes = [_u64]
        lib.pdo_flipped_bit_index.restype = _uint
        lib.pdo_flipped_bit_index.argtypes = [_u64]
        for name in ("pdo_coeff_fast", "pdo_coeff_slow"):
            f = getattr(lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [_uint, _dp, _u64, _dp]
        lib.pdo_decompose.restype = ctypes.c_int
        lib.pdo_decompose.argtypes = [_uint, _dp, _dp, _uint]
        lib.pdo_coeff_batch.restype = ctypes.c_int
        lib.pdo_coeff_batch.argtypes = [_uint, _dp, _u64p, _u64, _dp, _uint]
        lib.pdo_recompose.restype = ctypes.c_int
        lib.pdo_recompose.argtypes = [_uint, _dp, _dp]
        lib.pdo_matrix_seed.restype = _u64
        lib.pdo_matrix_seed.argtypes = [_u64, _uint, _uint]
        lib.pdo_random_matrix.restype = ctypes.c_int
        lib.pdo_random_matrix.argtypes = [_uint, _u64, _dp]
        self.lib = lib

    @staticmethod
    def _n(g: np.ndarray) -> int:
        return int(g.shape[0]).bit_length() - 1

    def xy_mask(self, n: int, nq: int) -> int:
        return int(self.lib.pdo_xy_mask(n, nq))

    def initial_phase(self, n: int, nq: int) -> int:
        return int(self.lib.pdo_initial_phase(n, nq))

    def coeff_fast(self, g, n: int) -> complex:
        g = _as_c128(g)
        out = np.zeros(2)
        if self.lib.pdo_coeff_fast(self._n(g), _ptr(g.view(np.float64)), n, _ptr(out)) != 0:
            raise ValueError("tensor number out of range")
        return complex(out[0], out[1])

    def coeff_slow(self, g, n: int) -> complex:
        g = _as_c128(g)
        out = np.zeros(2)
        if self.lib.pdo_coeff_slow(self._n(g), _ptr(g.view(np.float64)), n, _ptr(out)) != 0:
            raise ValueError("tensor number out of range")
        return complex(out[0], out[1])

    def decompose(self, g, threads: int = os.cpu_count() or 1) -> np.ndarray:
        g = _as_c128(g)
        nq = self._n(g)
        out = np.empty(4**nq, dtype=np.complex128)
        rc = self.lib.pdo_decompose(nq, _ptr(g.view(np.float64)), _ptr(out.view(np.float64)), threads)
        if rc != 0:
            raise ValueError("bad decomposition arguments")
        return out

    def coeff_batch(self, g, ns, threads: int = os.cpu_count() or 1) -> np.ndarray:
        g = _as_c128(g)
        ns = np.ascontiguousarray(ns, dtype=np.uint64)
        out = np.empty(ns.size, dtype=np.complex128)
        rc = self.lib.pdo_coeff_batch(self._n(g), _ptr(g.view(np.float64)), _ptr(ns, _u64p),
                                      ns.size, _ptr(out.view(np.float64)), threads)
        if rc != 0:
            raise ValueError("tensor number out of range")
        return out

    def recompose(self, coeffs) -> np.ndarray:
        c = np.ascontiguousarray(coeffs, dtype=np.complex128)
        nq = (int(c.size).bit_length() - 1) // 2
        out = np.empty((2**nq, 2**nq), dtype=np.complex128)
        if self.lib.pdo_recompose(nq, _ptr(c.view(np.float64)), _ptr(out.view(np.float64))) != 0:
            raise ValueError("bad coefficient count")
        return out

    def matrix_seed(self, seed: int, nq: int, rep: int) -> int:
        return int(self.lib.pdo_matrix_seed(seed, nq, rep))

    def random_matrix(self, nq: int, seed: int) -> np.ndarray:
        out = np.empty((2**nq, 2**nq), dtype=np.complex128)
        if self.lib.pdo_random_matrix(nq, seed, _ptr(out.view(np.float64))) != 0:
            raise ValueError("bad qubit count")
        return out


class Reference:
    """The reference's own C++ library (proj/src), via oracle/ref_harness.cpp."""

    def __init__(self, path: str = REF_SO):
        lib = ctypes.CDLL(path)
        lib.pdref_last_error.restype = ctypes.c_char_p
        lib.pdref_hardware_concurrency.restype = _uint
        lib.pdref_matrix_new.restype = ctypes.c_void_p
        lib.pdref_matrix_new.argtypes = [_uint, _dp]
        lib.pdref_matrix_random.restype = ctypes.c_void_p
        lib.pdref_matrix_random.argtypes = [_uint, _u64]
        lib.pdref_matrix_data.restype = _dp
        lib.pdref_matrix_data.argtypes = [ctypes.c_void_p]
        lib.pdref_matrix_free.argtypes = [ctypes.c_void_p]
        lib.pdref_matrix_seed.restype = _u64
        lib.pdref_matrix_seed.argtypes = [_u64, _uint, _uint]
        lib.pdref_random_matrix.argtypes = [_uint, _u64, _dp]
        lib.pdref_decompose_parallel.argtypes = [ctypes.c_void_p, _uint, _dp]
        lib.pdref_decompose_serial.argtypes = [ctypes.c_void_p, _dp]
        for name in ("pdref_coeff_fast", "pdref_coeff_slow", "pdref_oracle_kron"):
            getattr(lib, name).argtypes = [ctypes.c_void_p, _u64, _dp]
        lib.pdref_coeff_batch.argtypes = [ctypes.c_void_p, _u64p, _u64, _dp, _uint]
        lib.pdref_recompose.argtypes = [_uint, _dp, _dp]
        lib.pdref_format_double.argtypes = [ctypes.c_double, ctypes.c_char_p, _uint]
        lib.pdref_write_matrix_file.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int]
        lib.pdref_read_matrix_file.restype = ctypes.c_void_p
        lib.pdref_read_matrix_file.argtypes = [ctypes.c_char_p, ctypes.c_int]
        lib.pdref_matrix_qubits.restype = _uint
        lib.pdref_matrix_qubits.argtypes = [ctypes.c_void_p]
        lib.pdref_write_coefficients_file.restype = ctypes.c_longlong
        lib.pdref_write_coefficients_file.argtypes = [_uint, _dp, ctypes.c_char_p, ctypes.c_double]
        lib.pdref_read_coefficients_file.argtypes = [ctypes.c_char_p, ctypes.POINTER(_uint), _dp,
                                                     ctypes.c_ulonglong]
        self.lib = lib
        self.cores = int(lib.pdref_hardware_concurrency())

    def _check(self, rc: int) -> None:
        if rc != 0:
            msg = self.lib.pdref_last_error().decode()
            raise (ValueError if rc in (-1, -2, -4) else RuntimeError)(msg)

    class Matrix:
        def __init__(self, ref: "Reference", handle: int, nq: int):
            if not handle:
                raise ValueError(ref.lib.pdref_last_error().decode())
            self.ref, self.h, self.nq = ref, handle, nq

        def __del__(self):
            if getattr(self, "h", None):
                self.ref.lib.pdref_matrix_free(self.h)
                self.h = None

        def to_numpy(self) -> np.ndarray:
            d = 2**self.nq
            p = self.ref.lib.pdref_matrix_data(self.h)
            flat = np.ctypeslib.as_array(p, shape=(2 * d * d,))
            return flat.view(np.complex128).reshape(d, d).copy()

    def matrix(self, g) -> "Reference.Matrix":
        g = _as_c128(g)
        nq = int(g.shape[0]).bit_length() - 1
        return Reference.Matrix(self, self.lib.pdref_matrix_new(nq, _ptr(g.view(np.float64))), nq)

    def random_matrix_handle(self, nq: int, seed: int) -> "Reference.Matrix":
        return Reference.Matrix(self, self.lib.pdref_matrix_random(nq, seed), nq)

    def _h(self, g):
        return g if isinstance(g, Reference.Matrix) else self.matrix(g)

    def random_matrix(self, nq: int, seed: int) -> np.ndarray:
        out = np.empty((2**nq, 2**nq), dtype=np.complex128)
        self._check(self.lib.pdref_random_matrix(nq, seed, _ptr(out.view(np.float64))))
        return out

    def matrix_seed(self, seed: int, nq: int, rep: int) -> int:
        return int(self.lib.pdref_matrix_seed(seed, nq, rep))

    def decompose(self, g, threads: int | None = None) -> np.ndarray:
        m = self._h(g)
        out = np.empty(4**m.nq, dtype=np.complex128)
        self._check(self.lib.pdref_decompose_parallel(m.h, threads or self.cores,
                                                      _ptr(out.view(np.float64))))
        return out

    def decompose_serial(self, g) -> np.ndarray:
        m = self._h(g)
        out = np.empty(4**m.nq, dtype=np.complex128)
        self._check(self.lib.pdref_decompose_serial(m.h, _ptr(out.view(np.float64))))
        return out

    def _one(self, fn, g, n: int) -> complex:
        m = self._h(g)
        out = np.zeros(2)
        self._check(fn(m.h, n, _ptr(out)))
        return complex(out[0], out[1])

    def coeff_fast(self, g, n: int) -> complex:
        return self._one(self.lib.pdref_coeff_fast, g, n)

    def coeff_slow(self, g, n: int) -> complex:
        return self._one(self.lib.pdref_coeff_slow, g, n)

    def oracle_kron(self, g, n: int) -> complex:
        return self._one(self.lib.pdref_oracle_kron, g, n)

    def coeff_batch(self, g, ns, threads: int | None = None) -> np.ndarray:
        m = self._h(g)
        ns = np.ascontiguousarray(ns, dtype=np.uint64)
        out = np.empty(ns.size, dtype=np.complex128)
        self._check(self.lib.pdref_coeff_batch(m.h, _ptr(ns, _u64p), ns.size,
                                               _ptr(out.view(np.float64)), threads or self.cores))
        return out

    def recompose(self, coeffs) -> np.ndarray:
        c = np.ascontiguousarray(coeffs, dtype=np.complex128)
        nq = (int(c.size).bit_length() - 1) // 2
        out = np.empty((2**nq, 2**nq), dtype=np.complex128)
        self._check(self.lib.pdref_recompose(nq, _ptr(c.view(np.float64)), _ptr(out.view(np.float64))))
        return out

    # ---- the reference's file formats (io.cpp) ----
    def format_double(self, v: float) -> str:
        buf = ctypes.create_string_buffer(64)
        assert self.lib.pdref_format_double(v, buf, 64) == 0
        return buf.value.decode()

    def write_matrix(self, g, path: str, binary: bool) -> None:
        m = self._h(g)
        self._check(self.lib.pdref_write_matrix_file(m.h, path.encode(), int(binary)))

    def read_matrix(self, path: str, binary: bool) -> np.ndarray:
        h = self.lib.pdref_read_matrix_file(path.encode(), int(binary))
        if not h:
            raise ValueError(self.lib.pdref_last_error().decode())
        return Reference.Matrix(self, h, int(self.lib.pdref_matrix_qubits(h))).to_numpy()

    def write_coefficients(self, coeffs, path: str, threshold: float = 0.0) -> int:
        c = np.ascontiguousarray(coeffs, dtype=np.complex128)
        nq = (int(c.size).bit_length() - 1) // 2
        r = self.lib.pdref_write_coefficients_file(nq, _ptr(c.view(np.float64)), path.encode(), threshold)
        if r < 0:
            self._check(int(r))
        return int(r)

    def read_coefficients(self, path: str, max_qubits: int = 10) -> np.ndarray:
        nq = _uint(0)
        cap = 4**max_qubits
        out = np.zeros(cap, dtype=np.complex128)
        self._check(self.lib.pdref_read_coefficients_file(path.encode(), ctypes.byref(nq),
                                                          _ptr(out.view(np.float64)), cap))
        return out[: 4**nq.value].copy()


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def reference() -> Reference | None:
    """The compiled reference, or None when oracle/_ref was never built."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = Reference()
    return _ref


# ---- index algebra shared by tests (restated from SURVEY §0.1 / pauli.hpp) ----

def spread_bits(v: np.ndarray | int, nq: int):
    """Place bit t of v at bit 2t."""
    out = np.zeros_like(np.asarray(v, dtype=np.uint64))
    v = np.asarray(v, dtype=np.uint64)
    for t in range(nq):
        out |= ((v >> np.uint64(t)) & np.uint64(1)) << np.uint64(2 * t)
    return out


def xz_to_n(x, z, nq: int):
    """Tensor number of the string with X-mask x and Z-mask z: d_t = 2 z_t + (x_t ^ z_t)."""
    x = np.asarray(x, dtype=np.uint64)
    z = np.asarray(z, dtype=np.uint64)
    return spread_bits(x ^ z, nq) | (spread_bits(z, nq) << np.uint64(1))


def xmask_sample_indices(nq: int, xmasks) -> np.ndarray:
    """All tensor numbers whose X-mask is in xmasks, ascending (BASELINE.md §2 N=14 sample)."""
    z = np.arange(2**nq, dtype=np.uint64)
    ns = np.concatenate([xz_to_n(np.uint64(x), z, nq) for x in xmasks])
    return np.sort(ns)
