"""Device-side handles: operators, patch sets, vectors (plumbing over the C-ABI).

PyTorch supplies device memory and the current stream; the arithmetic is the
C-ABI library's.  Host objects (this package's or the reference's, duck-typed
on ``nrows, ncols, row_offsets, col_indices, values``) are uploaded once and
cached by identity.
"""

from __future__ import annotations

import ctypes
import weakref
from typing import Optional, Tuple

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda() -> None:
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_2402_12947_b200 needs a CUDA device (sm_100a): the hot path "
                           "has no CPU fallback")


def stream_handle() -> int:
    return torch().cuda.current_stream().cuda_stream


def _i64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _f64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def as_device_vector(x, n: Optional[int] = None, name: str = "vector"):
    """Return (tensor, host_array_or_None).  numpy -> fresh device copy."""
    t = torch()
    if isinstance(x, t.Tensor):
        if not x.is_cuda or x.dtype != t.float64:
            raise ValueError(f"{name} must be a CUDA float64 tensor or a numpy array")
        if not x.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if n is not None and x.shape != (n,):
            raise ValueError(f"dimension mismatch: expected {name} of length {n}, got {tuple(x.shape)}")
        return x, None
    arr = np.asarray(x, dtype=np.float64)
    if n is not None and arr.shape != (n,):
        raise ValueError(f"dimension mismatch: expected {name} of length {n}, got {arr.shape}")
    require_cuda()
    return t.from_numpy(np.ascontiguousarray(arr)).to("cuda", non_blocking=False), arr


class DeviceOperator:
    """Device copy of one CSR matrix (smg_operator)."""

    def __init__(self, m, with_transpose: bool = False):
        require_cuda()
        lib = _lib.load()
        self.nrows, self.ncols = int(m.nrows), int(m.ncols)
        ptr = np.ascontiguousarray(m.row_offsets, dtype=np.int64)
        col = np.ascontiguousarray(m.col_indices, dtype=np.int64)
        val = np.ascontiguousarray(m.values, dtype=np.float64)
        h = ctypes.c_void_p()
        _lib.check(lib.smg_operator_create(self.nrows, self.ncols, _i64(ptr), _i64(col), _f64(val),
                                           1 if with_transpose else 0, ctypes.byref(h)))
        self.handle = h
        self.with_transpose = with_transpose
        nr, nc, nnz, fz, db = (ctypes.c_int64() for _ in range(5))
        _lib.check(lib.smg_operator_info(h, ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(nnz),
                                         ctypes.byref(fz), ctypes.byref(db)))
        self.nnz = nnz.value
        self.first_zero_diag = fz.value
        self.device_bytes = db.value
        self._finalizer = weakref.finalize(self, lib.smg_operator_destroy, h)


class DeviceCorrection:
    """Device copy of a LocalCorrection (smg_correction)."""

    def __init__(self, op: DeviceOperator, correction):
        lib = _lib.load()
        idxs, facs = [], []
        for idx, factor in correction.regions:
            f = getattr(factor, "factor", factor)
            kind = getattr(factor, "kind", "cholesky")
            if kind != "cholesky":
                raise ValueError("local corrections must carry Cholesky factors (smoothers.py:195)")
            c, lower = f if isinstance(f, tuple) else (f, True)
            if not lower:
                raise ValueError("local corrections must carry lower Cholesky factors")
            idxs.append(np.asarray(idx, dtype=np.int64))
            facs.append(np.ascontiguousarray(c, dtype=np.float64))
        self.n_regions = len(idxs)
        roff = np.zeros(len(idxs) + 1, dtype=np.int64)
        np.cumsum([len(i) for i in idxs], out=roff[1:])
        dofs = np.concatenate(idxs) if idxs else np.zeros(0, dtype=np.int64)
        foff = np.zeros(len(facs) + 1, dtype=np.int64)
        np.cumsum([f.size for f in facs], out=foff[1:])
        flat = np.concatenate([f.ravel() for f in facs]) if facs else np.zeros(0)
        h = ctypes.c_void_p()
        _lib.check(lib.smg_correction_create(op.handle, self.n_regions, _i64(roff), _i64(dofs),
                                             _i64(foff), _f64(flat), ctypes.byref(h)))
        self.handle = h
        self.op = op
        nreg, cov, cpl, db = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_int64()
        _lib.check(lib.smg_correction_info(h, ctypes.byref(nreg), ctypes.byref(cov),
                                           ctypes.byref(cpl), ctypes.byref(db)))
        self.covered = cov.value
        self.coupled = bool(cpl.value)
        self.device_bytes = db.value
        self.n_global = int(correction.n_global)
        self._finalizer = weakref.finalize(self, lib.smg_correction_destroy, h)


_op_cache = {}
_corr_cache = {}


def _cached(cache, obj, make):
    key = id(obj)
    hit = cache.get(key)
    if hit is not None and hit[0]() is obj:
        return hit[1]
    val = make()
    try:
        ref = weakref.ref(obj, lambda _r, k=key: cache.pop(k, None))
    except TypeError:
        ref = (lambda o=obj: o)  # keeps obj alive; acceptable for non-weakrefable inputs
    cache[key] = (ref, val)
    return val


def device_operator(m, with_transpose: bool = False) -> DeviceOperator:
    """Upload (once) and return the device operator for a host CSR matrix."""
    key_cache = _op_cache
    op = _cached(key_cache, m, lambda: DeviceOperator(m, with_transpose))
    if with_transpose and not op.with_transpose:
        op = DeviceOperator(m, True)
        key_cache[id(m)] = (key_cache[id(m)][0], op)
    return op


def device_correction(a, correction) -> DeviceCorrection:
    """Device copy of ``correction`` bound to the operator ``a`` (its patch
    residuals are formed from a's rows, so the cache is keyed on both)."""
    n = int(getattr(a, "nrows"))
    if int(correction.n_global) != n:
        raise ValueError(f"correction size {int(correction.n_global)} does not match the "
                         f"{n}-row operator")
    op = device_operator(a)
    per_op = _cached(_corr_cache, correction, dict)
    hit = per_op.get(id(op))
    if hit is None or hit.op is not op:
        hit = DeviceCorrection(op, correction)
        per_op.clear()          # one operator per correction at a time (bounded)
        per_op[id(op)] = hit
    return hit


def _csr_result_to_host(lib, h):
    """Copy an smg_csr result to host arrays and free it."""
    try:
        nr, nc, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.smg_csr_info(h, ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(nnz)))
        ptr_ = np.empty(nr.value + 1, dtype=np.int64)
        col = np.empty(nnz.value, dtype=np.int64)
        val = np.empty(nnz.value, dtype=np.float64)
        _lib.check(lib.smg_csr_to_host(h, _i64(ptr_), _i64(col), _f64(val)))
        return nr.value, nc.value, ptr_, col, val
    finally:
        lib.smg_csr_destroy(h)


def galerkin(a, p):
    """``P^T (A P)`` on the device (smg_galerkin): (nrows, ncols, ptr, col, val)."""
    lib = _lib.load()
    oa = device_operator(a)
    op = device_operator(p, with_transpose=True)
    h = ctypes.c_void_p()
    _lib.check(lib.smg_galerkin(oa.handle, op.handle, ctypes.byref(h), stream_handle()))
    return _csr_result_to_host(lib, h)


def matmul(x, y):
    """``X Y`` on the device (smg_matmul): (nrows, ncols, ptr, col, val)."""
    lib = _lib.load()
    ox, oy = device_operator(x), device_operator(y)
    h = ctypes.c_void_p()
    _lib.check(lib.smg_matmul(ox.handle, oy.handle, ctypes.byref(h), stream_handle()))
    return _csr_result_to_host(lib, h)


def ptr(t) -> int:
    return int(t.data_ptr())
