"""CPU-side checks of the C-ABI boundary: the library loads without a GPU and
exports every symbol include/usbs_b200.h declares (no compute calls)."""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "usbs_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(usbs_[a-z0-9_]+)\s*\(", text)
    return sorted(set(n for n in names if n not in ("usbs_rng_fill_fn",)))


def test_header_declares_entry_points():
    names = declared_symbols()
    for must in ("usbs_ctx_create", "usbs_problem_create", "usbs_op_apply", "usbs_lanczos_top"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2312_11801_b200 import _native

    if not _native.LIB_PATH.exists():
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing
    # every binding in _native refers to a declared symbol
    assert set(_native.PROTOS) <= set(declared_symbols())
    assert lib.usbs_abi_version() == 1


def test_status_mapping_matches_reference_exceptions():
    from paper_2312_11801_b200 import _native
    from paper_2312_11801_b200.errors import ConditioningError, EmptyBasisError, NumericError, StepFailureError

    if not _native.LIB_PATH.exists():
        pytest.skip("library not built")
    _native.load()
    for code, exc in ((1, ValueError), (2, ValueError), (3, NumericError), (4, ConditioningError),
                      (5, StepFailureError), (6, EmptyBasisError), (7, RuntimeError)):
        with pytest.raises(exc):
            _native.check(code, "probe")
    _native.check(0)


def test_make_test_matrix_bit_exact_with_numpy():
    """usbs_make_test_matrix (host-only entry point, callable without a GPU)
    equals make_test_matrix (sketch.py:25-27) = numpy's legacy
    RandomState(seed & 0x7FFFFFFF).standard_normal((n, r)) bit for bit, for
    row slices (the sharded sketch) and seeds above 2^31."""
    import numpy as np

    from paper_2312_11801_b200 import _native
    if not _native.LIB_PATH.exists():
        pytest.skip("library not built (run __graft_entry__.build())")
    from paper_2312_11801_b200.solver import make_test_matrix_rows
    for n, r, seed, r0, r1 in ((1000, 10, 5, 0, 1000), (1001, 7, 2**31 + 17, 3, 900), (1, 1, 0, 0, 1),
                               (0, 5, 1, 0, 0), (20000, 20, 123456789, 100, 19999)):
        want = np.random.RandomState(int(seed) & 0x7FFFFFFF).standard_normal((n, r))[r0:r1]
        assert np.array_equal(make_test_matrix_rows(n, r, seed, r0, r1), want)
    with pytest.raises(ValueError):
        make_test_matrix_rows(10, 2, 0, 5, 11)
