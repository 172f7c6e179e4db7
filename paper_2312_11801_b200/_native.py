"""ctypes binding of the C ABI in include/usbs_b200.h.

The product path has no CPU fallback: if ``libusbs_b200.so`` is missing or
no CUDA device is present, importing the device layer raises.  Status codes
are mapped onto the reference's exception types (include/usbs_b200.h).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import (
    ConditioningError,
    EmptyBasisError,
    NumericError,
    StepFailureError,
)

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libusbs_b200.so"

_p = C.c_void_p
_pd = C.POINTER(C.c_double)
_pi = C.POINTER(C.c_int)
_i64 = C.c_int64
_i32 = C.c_int

RNG_FILL = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64)

# name -> (restype, argtypes)
PROTOS = {
    "usbs_abi_version": (C.c_int, []),
    "usbs_last_error": (C.c_char_p, []),
    "usbs_ctx_create": (_i32, [_i32, _p, C.POINTER(_p)]),
    "usbs_ctx_destroy": (_i32, [_p]),
    "usbs_ctx_sync": (_i32, [_p]),
    "usbs_ctx_launches": (_i64, [_p]),
    "usbs_memcpy_h2d": (_i32, [_p, _p, _p, _i64]),
    "usbs_memcpy_d2h": (_i32, [_p, _p, _p, _i64]),
    "usbs_problem_create": (_i32, [_p, _i64, _i64, _p, _p, _p, _i64, _p, _p, _p, _p, _i32, C.POINTER(_p)]),
    "usbs_problem_create_shard": (_i32, [_p, _i64, _i64, _i64, _p, _p, _p, _i64, _p, _p, _p, _p, _i32,
                                         C.POINTER(_p)]),
    "usbs_problem_destroy": (_i32, [_p]),
    "usbs_problem_info": (_i32, [_p, C.POINTER(_i64), C.POINTER(_i64), _pi, _pi]),
    "usbs_slack_assemble": (_i32, [_p, _p, _p]),
    "usbs_problem_set_kron": (_i32, [_p, _p, _i32, _p, _p, C.c_double]),
    "usbs_lz_step_finish": (_i32, [_p, _i32, _i32, _p, _p, _p, _p, _p, _p, _i64, _i64, _p, _i64]),
    "usbs_lz_restart_h": (_i32, [_p, _i32, _i32, _p, _p]),
    "usbs_op_apply": (_i32, [_p, _p, _i32, _p, _i64, _i32, _p, _i64, _p]),
    "usbs_lanczos_top": (_i32, [_p, _p, _i32, _i32, _i32, _i32, C.c_double, _p, RNG_FILL, _p,
                                 _pd, _p, _i64, _pd, _pi, _pi, _pd, _pi, _pi]),
    "usbs_small_eigh": (_i32, [_p, _i32, _p, _p, _p]),
    "usbs_lanczos_profile": (_i32, [_p, C.POINTER(C.c_uint64), _i32]),
    "usbs_lanczos_plan": (_i32, [_p, _p, _i32, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "usbs_ipm_solve": (_i32, [_p, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p]),
    "usbs_ipm_state_len": (_i32, [_i32]),
    "usbs_loop_begin": (_i32, [_p]),
    "usbs_loop_end": (_i32, [_p, _p, C.c_double, _i32, _p]),
    "usbs_loop_abort": (_i32, [_p]),
    "usbs_ipm_profile": (_i32, [_p, C.POINTER(C.c_uint64), _i32]),
    "usbs_cons_image": (_i32, [_p, _p, _p, _i64, _i32, _p, _i32, C.c_double, _p, C.c_double, _p, _p]),
    "usbs_cons_compressed": (_i32, [_p, _p, _p, _i64, _i32, C.c_double, _p, _p, C.c_double, _p, _p,
                                    C.c_double, _p]),
    "usbs_rowgemm": (_i32, [_p, _i64, _p, _i64, _i32, _p, _i64, _i32, _p, C.c_double, C.c_double, _p, _i64, _p,
                            _i64]),
    "usbs_gram": (_i32, [_p, _i64, _p, _i64, _i32, _p, _i64, _i32, _p, _i32]),
    "usbs_wcoldot": (_i32, [_p, _i64, _p, _i64, _p, _i64, _i32, _p, _p]),
    "usbs_dense_update": (_i32, [_p, _i64, _p, C.c_double, _p, _i64, _i32, _p]),
    "usbs_vec": (_i32, [_p, _i32, _i64, _p, _p, _p, _p, _p, C.c_double, C.c_double, _p, _p]),
    "usbs_pivchol": (_i32, [_p, _i32, _p, C.c_double, _p, _p, _p]),
    "usbs_svec": (_i32, [_p, _i32, _p, C.c_double, _p]),
    "usbs_gather": (_i32, [_p, _i64, _p, _p, _p]),
    "usbs_gather_rows": (_i32, [_p, _i64, _i32, _p, _p, _i64, _p, _i64]),
    "usbs_cons_adjoint_apply": (_i32, [_p, _p, _p, _p, _i64, _i32, _p, _i64, _p]),
    "usbs_cons_adjoint_values": (_i32, [_p, _p, _p, _p]),
    "usbs_problem_pattern": (_i32, [_p, _p, _p, _p]),
    "usbs_cons_image_dense": (_i32, [_p, _p, _p, _i64, _p]),
    "usbs_cons_compressed_rows": (_i32, [_p, _p, _p, _i64, _i32, _p, _i64]),
    "usbs_perm_rows": (_i32, [_p, _i32, _p, _p, _p, _p]),
    "usbs_maxcut_round": (_i32, [_p, _i64, _i64, _p, _p, _p, _p, _i64, _i32, _pd, _pi, _p]),
    "usbs_make_test_matrix": (_i32, [_i64, _i64, _i32, _i64, _i64, _p]),
}

# VecOp codes (csrc/usbs_book.cu)
VOP_W, VOP_PROJN, VOP_AXPBY, VOP_NUNEXT, VOP_CAND, VOP_RESID, VOP_DOT, VOP_MINI, VOP_RELU, VOP_DOTAFF, VOP_PSIWY, \
    VOP_PSIWW = range(12)

# symbols declared in include/usbs_b200.h that must be exported (checked by tests)
_lib = None


def load(path: Path | None = None):
    """Load (once) and return the shared library with prototypes set."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(path or os.environ.get("USBS_LIB", LIB_PATH))
    if not path.exists():
        raise RuntimeError(f"libusbs_b200.so not built at {path}; run __graft_entry__.build() "
                           "(the device path has no CPU fallback)")
    lib = C.CDLL(str(path))
    for name, (res, args) in PROTOS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


class UsbsCudaError(RuntimeError):
    pass


def check(status: int, what: str = ""):
    if status == 0:
        return
    msg = (_lib.usbs_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status in (1, 2):
        raise ValueError(text)
    if status == 3:
        raise NumericError(text)
    if status == 4:
        raise ConditioningError(text)
    if status == 5:
        raise StepFailureError(text)
    if status == 6:
        raise EmptyBasisError(text)
    raise UsbsCudaError(f"status {status}: {text}")


def ptr(t) -> int:
    """Device/host address of a torch tensor or numpy array."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data
