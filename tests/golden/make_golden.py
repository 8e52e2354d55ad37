"""Generate tests/golden/*.npz from the REFERENCE itself.

Run in the build container, where /root/reference exists and oracle/Makefile
has compiled the reference's own pybind module (proj/bindings/module.cpp) and
C++ core (proj/src) into oracle/_ref/:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures are plain arrays (inputs + the reference's outputs), so the GPU
box — which has no /root/reference — can check against them.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, ROOT)

import _paulidecomp as ref  # noqa: E402  (the reference's own module)
from oracle import oracle as O  # noqa: E402

ACCEPT_SEED = 20260823  # proj/tests/acceptance.cpp:30


def normal_matrix(rng, nq):  # proj/tests/python/test_smoke.py:32-34
    d = 2**nq
    return rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))


def main() -> None:
    R = O.reference()
    out = {}

    # KAT proj/tests/test_decompose.cpp:69-77, test_smoke.py:57-65
    kat = np.array([[1, 2], [3, 4]], dtype=complex)
    out["kat_matrix"] = kat
    out["kat_coeffs"] = ref.decompose(kat)

    # numpy N(0,1) matrices N=1..6 (test_smoke.py construction); N=6 is BASELINE config C1
    for nq in range(1, 7):
        g = normal_matrix(np.random.default_rng(1234 + nq), nq)
        out[f"normal{nq}_matrix"] = g
        out[f"normal{nq}_coeffs"] = ref.decompose(g)
        out[f"normal{nq}_serial"] = ref.decompose(g, serial=True)

    # reference random_matrix (bench.cpp:48-58) with acceptance seeds, N=1..6
    for nq in range(1, 7):
        seed = R.matrix_seed(ACCEPT_SEED, nq, 0)
        g = R.random_matrix(nq, seed)
        out[f"unif{nq}_seed"] = np.uint64(seed)
        out[f"unif{nq}_matrix"] = g
        out[f"unif{nq}_coeffs"] = ref.decompose(g, threads=4)

    # N=14 generator pin: first and last 4096 elements + 4096 scattered ones of
    # random_matrix(14, seed), plus 64 reference coeff_fast values at seeded n
    seed14 = R.matrix_seed(ACCEPT_SEED, 14, 0)
    h = R.random_matrix_handle(14, seed14)
    g14 = h.to_numpy().reshape(-1)
    rng = np.random.default_rng(14)
    idx = np.sort(rng.choice(g14.size, 4096, replace=False)).astype(np.uint64)
    out["unif14_seed"] = np.uint64(seed14)
    out["unif14_head"] = g14[:4096].copy()
    out["unif14_tail"] = g14[-4096:].copy()
    out["unif14_idx"] = idx
    out["unif14_at_idx"] = g14[idx.astype(np.int64)].copy()
    ns14 = np.sort(rng.choice(4**14, 64, replace=False)).astype(np.uint64)
    out["unif14_ns"] = ns14
    out["unif14_ns_coeffs"] = R.coeff_batch(h, ns14)
    del g14, h

    # Hermitian N=4 (test_decompose.cpp:36-45 construction on random_matrix)
    g = R.random_matrix(4, 99)
    for j in range(16):
        for i in range(j + 1):
            hval = 0.5 * (g[j, i] + np.conj(g[i, j]))
            g[j, i] = hval
            g[i, j] = np.conj(hval)
    out["herm4_matrix"] = g
    out["herm4_coeffs"] = ref.decompose(g)

    # batched strings at N=8 (BASELINE config C2 shape, scaled down): reference coefficient()
    g = normal_matrix(np.random.default_rng(808), 8)
    ns = np.random.default_rng(809).integers(0, 4**8, 512).astype(np.uint64)
    out["batch8_matrix"] = g
    out["batch8_ns"] = ns
    out["batch8_coeffs"] = np.array([ref.coefficient(g, int(n)) for n in ns])

    # non-finite elements: the reference multiplies lambda * a[...] as std::complex<double>
    # (decompose.cpp:40), so 0 * inf terms are NaN; inf / -inf / NaN sprinkled over seeded N(0,1)
    # matrices N=1..6, with the reference's decompose (both drivers), coefficient(slow) and
    # recompose of the result
    kat_nf = np.array([[1, np.inf], [3, 4]], dtype=complex)
    out["nfkat_matrix"] = kat_nf
    out["nfkat_coeffs"] = ref.decompose(kat_nf)
    specials = np.array([np.inf, -np.inf, np.nan, 0.0, -0.0])
    rng = np.random.default_rng(4040)
    for k, nq in enumerate((1, 1, 2, 2, 3, 3, 4, 5, 6)):
        g = normal_matrix(rng, nq)
        for _ in range(int(rng.integers(1, 4))):
            i = int(rng.integers(0, 4**nq))
            part = g.real if rng.random() < 0.5 else g.imag
            part.flat[i] = rng.choice(specials)
        out[f"nf{k}_matrix"] = g
        out[f"nf{k}_coeffs"] = ref.decompose(g)
        out[f"nf{k}_serial"] = ref.decompose(g, serial=True)
        out[f"nf{k}_slow"] = np.array([ref.coefficient(g, n, slow=True) for n in range(min(4**nq, 64))])
        out[f"nf{k}_recomposed"] = ref.recompose(out[f"nf{k}_coeffs"])

    # label helpers (module.cpp:108-114)
    labels = ["I", "X", "Y", "Z", "XY", "IX", "ZZ", "IXZY", "YYYYY", "ZIXYIZ"]
    out["labels"] = np.array(labels)
    out["label_index"] = np.array([ref.label_to_index(s, len(s)) for s in labels], dtype=np.uint64)
    ks = np.arange(0, 300, dtype=np.uint64)
    out["gray_k"] = ks
    out["gray_code"] = np.array([ref.gray_code(int(k)) for k in ks], dtype=np.uint64)
    out["flipped_bit"] = np.array([ref.flipped_bit_index(int(k)) for k in ks], dtype=np.uint64)
    out["xy_mask_n"] = np.arange(256, dtype=np.uint64)
    out["xy_mask_4"] = np.array([ref.xy_mask(int(n), 4) for n in range(256)], dtype=np.uint64)

    path = os.path.join(HERE, "reference_vectors.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
