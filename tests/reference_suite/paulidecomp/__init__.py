"""`paulidecomp` resolved to the B200 package: the reference's package re-export
(proj/python/paulidecomp/__init__.py) over `paper_2401_16378_b200` instead of its own CPU
extension, as INTEGRATION.md §2b describes. Test infrastructure: tests/test_reference_suite_gpu.py
puts this directory first on PYTHONPATH and runs the reference's own pytest file unchanged."""
from paper_2401_16378_b200 import (  # noqa: F401
    FormatError,
    __version__,
    coefficient,
    decompose,
    flipped_bit_index,
    gray_code,
    index_to_label,
    label_to_index,
    oracle_coefficient,
    recompose,
    xy_mask,
)

__all__ = [
    "FormatError", "__version__", "coefficient", "decompose", "flipped_bit_index", "gray_code",
    "index_to_label", "label_to_index", "oracle_coefficient", "recompose", "xy_mask",
]
