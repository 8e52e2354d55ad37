"""Pauli-string decomposition of dense complex matrices on NVIDIA B200 (sm_100a).

Drop-in for the reference package ``paulidecomp`` (proj/python/paulidecomp/__init__.py):
the same public names, argument meanings and exceptions, served by hand-written CUDA
kernels through the C ABI in ``include/pd_api.h``:

    decompose(matrix, threads=1, serial=False, path="gray", out=None, devices=None)
    coefficient(matrix, n | label, slow=False)
    oracle_coefficient(matrix, n | label)
    recompose(coefficients)
    gray_code, flipped_bit_index, xy_mask, label_to_index, index_to_label, FormatError

B200 additions: ``coefficients`` (batched strings), ``device`` (stream-ordered entry points
on device pointers), ``sharding`` (X-mask sharding over GPUs with NCCL), ``launch_count``, and
the reference's file formats (``read_matrix``/``write_matrix``/``read_coefficients``/
``write_coefficients``/``format_double``) with ``decompose_file`` feeding the GPU directly;
the ``pdb200`` executable mirrors the reference CLI's decompose/recompose/coeff.

There is no CPU fallback: importing this package without its compiled extension raises,
and every compute call without an sm_100 GPU raises RuntimeError.
"""
from __future__ import annotations

import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))

try:
    from . import _paulidecomp as _ext  # noqa: F401  (the compiled module)
except ImportError as exc:  # pragma: no cover - exercised only on a broken build
    raise ImportError(
        "paper_2401_16378_b200: the CUDA extension is not built "
        f"({exc}); run `python -c 'import __graft_entry__ as g; g.build()'` "
        "or `make -C paper_2401_16378_b200/csrc`. There is no CPU fallback."
    ) from exc

from ._paulidecomp import (  # noqa: E402
    FormatError,
    __version__,
    coefficient,
    coefficients,
    decompose,
    decompose_file,
    device,
    format_double,
    flipped_bit_index,
    fp64_add_probe,
    gray_code,
    index_to_label,
    label_to_index,
    launch_count,
    matrix_seed,
    oracle_coefficient,
    read_coefficients,
    random_matrix,
    read_matrix,
    recompose,
    set_device,
    write_coefficients,
    write_matrix,
    xy_mask,
)

LIBRARY_PATH = _os.path.join(_HERE, "libpd_b200.so")

__all__ = [
    "FormatError",
    "__version__",
    "coefficient",
    "coefficients",
    "decompose",
    "decompose_file",
    "device",
    "format_double",
    "flipped_bit_index",
    "fp64_add_probe",
    "gray_code",
    "index_to_label",
    "label_to_index",
    "launch_count",
    "matrix_seed",
    "oracle_coefficient",
    "read_coefficients",
    "random_matrix",
    "read_matrix",
    "recompose",
    "set_device",
    "write_coefficients",
    "write_matrix",
    "xy_mask",
    "LIBRARY_PATH",
]
