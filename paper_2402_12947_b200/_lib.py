"""ctypes binding of the in-tree C-ABI library (include/simplexmg_b200.h).

The library is the only compute path: there is no CPU fallback.  Importing
this module never needs a GPU (the CPU test suite checks the exported
symbols); every compute entry point fails loudly if the library or a CUDA
device is missing.
"""

from __future__ import annotations

import ctypes
import os
import re

from . import build_lib

_i64 = ctypes.c_int64
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_intp = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p
_pp = ctypes.POINTER(ctypes.c_void_p)

SMG_OK = 0
SMG_ERR_INVALID = 1
SMG_ERR_DIMENSION = 2
SMG_ERR_CUDA = 3
SMG_ERR_ZERO_DIAGONAL = 4
SMG_ERR_INDEFINITE = 5
SMG_ERR_UNSUPPORTED = 6
SMG_ERR_POINT_LOCATION = 7
SMG_ERR_NOT_SPD = 8

# name -> (restype, argtypes); mirrors include/simplexmg_b200.h
PROTOTYPES = {
    "smg_abi_version": (ctypes.c_int, []),
    "smg_last_error": (ctypes.c_char_p, []),
    "smg_device_info": (ctypes.c_int, [_intp, _i64p, _intp, _intp]),
    "smg_operator_create": (ctypes.c_int, [_i64, _i64, _i64p, _i64p, _f64p, ctypes.c_int, _pp]),
    "smg_operator_destroy": (ctypes.c_int, [_vp]),
    "smg_operator_info": (ctypes.c_int, [_vp, _i64p, _i64p, _i64p, _i64p, _i64p]),
    "smg_operator_layout": (ctypes.c_int, [_vp, _intp, _intp]),
    "smg_operator_set_layout": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int]),
    "smg_spmv": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "smg_residual": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "smg_spmv_transpose": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "smg_prolong_add": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "smg_chebyshev_smooth": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, ctypes.c_double,
                                            ctypes.c_double, _vp, _vp]),
    "smg_smoother_step": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, ctypes.c_int, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, _vp]),
    "smg_correction_create": (ctypes.c_int, [_vp, _i64, _i64p, _i64p, _i64p, _f64p, _pp]),
    "smg_correction_destroy": (ctypes.c_int, [_vp]),
    "smg_correction_info": (ctypes.c_int, [_vp, _i64p, _i64p, _intp, _i64p]),
    "smg_apply_local_correction": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "smg_local_correct": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "smg_combined_smooth": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_double, ctypes.c_double, _vp, _vp]),
    "smg_hierarchy_create": (ctypes.c_int, [ctypes.c_int, _pp, _pp, _pp, _intp, _intp, _f64p,
                                            _f64p, _i64, _f64p, ctypes.c_int, _pp]),
    "smg_hierarchy_destroy": (ctypes.c_int, [_vp]),
    "smg_hierarchy_set_graphs": (ctypes.c_int, [_vp, ctypes.c_int]),
    "smg_hierarchy_set_option": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int]),
    "smg_hierarchy_launches_per_vcycle": (ctypes.c_int, [_vp, _i64p]),
    "smg_coarse_solve": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "smg_vcycle": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "smg_vcycle_host": (ctypes.c_int, [_vp, _f64p, _f64p, _vp]),
    "smg_vcycle_host_many": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp]),
    "smg_solve_stationary": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_double, ctypes.c_int,
                                            _f64p, _intp, _vp]),
    "smg_cg": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                              _f64p, _intp, _i64p, _f64p, _vp]),
    "smg_dot": (ctypes.c_int, [_i64, _vp, _vp, _f64p, _vp]),
    "smg_galerkin": (ctypes.c_int, [_vp, _vp, _pp, _vp]),
    "smg_matmul": (ctypes.c_int, [_vp, _vp, _pp, _vp]),
    "smg_csr_info": (ctypes.c_int, [_vp, _i64p, _i64p, _i64p]),
    "smg_csr_to_host": (ctypes.c_int, [_vp, _i64p, _i64p, _f64p]),
    "smg_csr_destroy": (ctypes.c_int, [_vp]),
    "smg_dense_cholesky": (ctypes.c_int, [_i64, _f64p, _f64p, _i64p, _vp]),
    "smg_cholesky_inverse": (ctypes.c_int, [_i64, _f64p, _f64p, _vp]),
    "smg_assemble_poisson": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _i64, _f64p, _i64, _i64p,
                                            _i64p, _i64, _i64p, _i64, _f64p, _f64p, ctypes.c_int,
                                            _pp, _i64p, _vp]),
    "smg_assemble_elements": (ctypes.c_int, [_i64, _i64, ctypes.c_int, _i64p, _f64p, _i64p, _i64,
                                             _pp, _vp]),
    "smg_patch_factor": (ctypes.c_int, [_vp, _i64, _i64p, _i64p, _f64p, _i64p, _i64p, _vp]),
    "smg_prolongation_build": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _i64, _f64p, _i64, _f64p,
                                              _f64p, _i64p, _i64, ctypes.c_int, _f64p, _f64p,
                                              _f64p, _i64p, _i64p, ctypes.c_double,
                                              ctypes.c_double, _pp, _i64p, _vp]),
}

_lib = None


class SmgError(RuntimeError):
    """A C-ABI call failed; ``code`` is the SMG_ERR_* value."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def library_path() -> str:
    return build_lib.LIB


def header_symbols() -> list:
    """Function names declared in include/simplexmg_b200.h."""
    with open(build_lib.HEADER) as f:
        text = f.read()
    return re.findall(r"^\s*SMG_API\s+(?:int|const char \*)\s*(smg_\w+)\s*\(", text, flags=re.M)


def load(build_if_missing: bool = True):
    """Load the shared library (building it in-tree if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    # SMG_LIB: an alternative in-tree build of the same C-ABI (compile-time
    # A/B variants, tools/build_variant.py); default: the product library
    path = os.environ.get("SMG_LIB", build_lib.LIB)
    if not os.path.exists(path):
        if not build_if_missing:
            raise RuntimeError(f"{path} is missing: run `python -m paper_2402_12947_b200.build_lib`")
        build_lib.build()
    lib = ctypes.CDLL(path)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != SMG_OK:
        msg = load().smg_last_error().decode(errors="replace")
        raise SmgError(rc, msg)
