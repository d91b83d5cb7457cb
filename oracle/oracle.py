"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the simplexmg combined-smoother hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module.
It is the checker, never the product: ``paper_2402_12947_b200`` does not
import it and has no CPU fallback.

This is a numpy + plain-C restatement of the reference algorithm
(``/root/reference/pkg/src/simplexmg``; paths below are relative to
``/root/reference/pkg/src/simplexmg``):

* elementwise work is numpy in exactly the reference's expression order, so
  it rounds identically;
* sparse products call ``smg_oracle.c`` (row-sequential, no FMA), which is
  bit-identical to scipy's ``csr_matvec`` / ``csc_matvec`` as the reference
  calls them;
* dense Cholesky solves (LAPACK ``dpotrs`` in the reference) are sequential
  substitutions with the reference's own factor; they agree to ~1e-15
  relative, pinned by ``tests/golden``.

Objects are duck-typed against the reference's data model: a matrix has
``nrows, ncols, row_offsets, col_indices, values``; a level has ``a``,
``prolongation.matrix``, ``smoother`` (``kind, sweeps, lambda_max,
lambda_min_fraction``), ``local_correction.regions`` as ``(idx, factor)``
with ``factor.factor == (c, lower)``; a hierarchy has ``levels`` and
``coarse_factor``.  Reference objects and ``paper_2402_12947_b200`` host
objects both fit.

Parity status: PINNED -- tests/test_oracle_golden.py checks every function
here against vectors produced by the reference itself
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Callable, List, Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libsmg_oracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile smg_oracle.c with oracle/Makefile (gcc; no GPU needed)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "smg_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_csr_matvec.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.oracle_csr_matvec_rows.argtypes = [ctypes.c_int64, _i64p, _i64p, _i64p, _f64p,
                                             _f64p, _f64p]
        L.oracle_csrT_matvec.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.oracle_chol_solve.argtypes = [ctypes.c_int64, _f64p, _f64p]
        L.oracle_patch_solves.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, _f64p]
        L.oracle_spgemm.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i64p, _f64p,
                                    _i64p, _i64p, _f64p, _i64p, _i64p, _f64p]
        L.oracle_dot.argtypes = [ctypes.c_int64, _f64p, _f64p]
        L.oracle_dot.restype = ctypes.c_double
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def _p(a, t):
    return a.ctypes.data_as(t)


# --------------------------------------------------------------------------
# sparse primitives

class _Csr:
    """int64/f64 contiguous copy of a CSR matrix (+ lazily its transpose)."""

    def __init__(self, m):
        self.nrows, self.ncols = int(m.nrows), int(m.ncols)
        self.ptr = np.ascontiguousarray(m.row_offsets, dtype=np.int64)
        self.col = np.ascontiguousarray(m.col_indices, dtype=np.int64)
        self.val = np.ascontiguousarray(m.values, dtype=np.float64)
        self._t = None
        self._diag = None

    def transpose(self):
        """CSR(P^T) with fine indices ascending in every row (stable sort)."""
        if self._t is None:
            rows = np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.ptr))
            order = np.argsort(self.col, kind="stable")
            tcol = rows[order]
            tval = self.val[order]
            counts = np.bincount(self.col, minlength=self.ncols)
            tptr = np.zeros(self.ncols + 1, dtype=np.int64)
            np.cumsum(counts, out=tptr[1:])
            self._t = (tptr, np.ascontiguousarray(tcol), np.ascontiguousarray(tval))
        return self._t

    def diagonal(self):
        """A.diagonal() (sparse.py:123-124): explicit entry or 0.0."""
        if self._diag is None:
            d = np.zeros(min(self.nrows, self.ncols))
            rows = np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.ptr))
            hit = rows == self.col
            d[rows[hit]] = self.val[hit]
            self._diag = d
        return self._diag


_cache = {}


def _csr(m) -> _Csr:
    key = id(m)
    hit = _cache.get(key)
    if hit is None or hit[0] is not m:
        hit = (m, _Csr(m))
        _cache[key] = hit
    return hit[1]


def spmv(a, x: np.ndarray) -> np.ndarray:
    """``a @ x`` (sparse.py:135-140 -> scipy csr_matvec), bit-identical."""
    c = _csr(a)
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape != (c.ncols,):
        raise ValueError(f"dimension mismatch: matrix is {c.nrows}x{c.ncols}, vector has length {x.shape}")
    y = np.empty(c.nrows)
    lib().oracle_csr_matvec(c.nrows, _p(c.ptr, _i64p), _p(c.col, _i64p), _p(c.val, _f64p),
                            _p(x, _f64p), _p(y, _f64p))
    return y


def spmv_rows(a, rows: np.ndarray, x: np.ndarray) -> np.ndarray:
    """``(a @ x)[rows]`` with the same per-row arithmetic."""
    c = _csr(a)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(len(rows))
    lib().oracle_csr_matvec_rows(len(rows), _p(rows, _i64p), _p(c.ptr, _i64p),
                                 _p(c.col, _i64p), _p(c.val, _f64p), _p(x, _f64p),
                                 _p(y, _f64p))
    return y


def spmv_transpose(p, r: np.ndarray) -> np.ndarray:
    """``p.to_scipy().T @ r`` (mg.py:142 -> scipy csc_matvec), bit-identical."""
    c = _csr(p)
    tptr, tcol, tval = c.transpose()
    r = np.ascontiguousarray(r, dtype=np.float64)
    if r.shape != (c.nrows,):
        raise ValueError(f"residual length {r.shape} does not match fine size {c.nrows}")
    y = np.empty(c.ncols)
    lib().oracle_csrT_matvec(c.ncols, _p(tptr, _i64p), _p(tcol, _i64p), _p(tval, _f64p),
                             _p(r, _f64p), _p(y, _f64p))
    return y


def diagonal(a) -> np.ndarray:
    return _csr(a).diagonal()


def _spgemm_arrays(nrows, ncols, xptr, xcol, xval, yptr, ycol, yval):
    ptr = np.zeros(nrows + 1, dtype=np.int64)
    args = [_p(np.ascontiguousarray(t, dtype=dt), tp)
            for t, dt, tp in ((xptr, np.int64, _i64p), (xcol, np.int64, _i64p),
                              (xval, np.float64, _f64p), (yptr, np.int64, _i64p),
                              (ycol, np.int64, _i64p), (yval, np.float64, _f64p))]
    keep = [np.ascontiguousarray(t) for t in (xptr, xcol, xval, yptr, ycol, yval)]  # noqa: F841
    lib().oracle_spgemm(nrows, ncols, *args, _p(ptr, _i64p), None, None)
    col = np.empty(int(ptr[-1]), dtype=np.int64)
    val = np.empty(int(ptr[-1]), dtype=np.float64)
    lib().oracle_spgemm(nrows, ncols, *args, _p(ptr, _i64p), _p(col, _i64p), _p(val, _f64p))
    return ptr, col, val


def spgemm(x, y):
    """``x @ y`` for CSR x, y (scipy csr_matmat order, explicit zeros dropped,
    columns sorted); returns (row_offsets, col_indices, values)."""
    a, b = _csr(x), _csr(y)
    if a.ncols != b.nrows:
        raise ValueError(f"dimension mismatch: {a.nrows}x{a.ncols} @ {b.nrows}x{b.ncols}")
    return _spgemm_arrays(a.nrows, b.ncols, a.ptr, a.col, a.val, b.ptr, b.col, b.val)


def galerkin(p, a):
    """Galerkin coarse operator ``p.T @ (a @ p)`` (sparse.py:147-154) as CSR arrays.

    scipy forms ``a @ p`` with csr_matmat, then ``p.T @ M`` as a CSC product
    whose column c accumulates ``M[i,c] * P[i,k]`` over fine rows i ascending;
    the same sums arise from CSR(P^T) @ M with CSR(P^T) listing fine rows
    ascending (multiplication commutes; the addition order is identical)."""
    pc, ac = _csr(p), _csr(a)
    if ac.ncols != pc.nrows or ac.nrows != pc.nrows:
        raise ValueError(f"dimension mismatch: a is {ac.nrows}x{ac.ncols}, p is {pc.nrows}x{pc.ncols}")
    mptr, mcol, mval = _spgemm_arrays(ac.nrows, pc.ncols, ac.ptr, ac.col, ac.val,
                                      pc.ptr, pc.col, pc.val)
    tptr, tcol, tval = pc.transpose()
    return _spgemm_arrays(pc.ncols, pc.ncols, tptr, tcol, tval, mptr, mcol, mval)


# --------------------------------------------------------------------------
# dense factor solves (sparse.py:214-231)

def _factor_array(factor) -> np.ndarray:
    f = getattr(factor, "factor", factor)
    if isinstance(f, tuple):
        c, lower = f
        if not lower:
            raise ValueError("oracle expects lower Cholesky factors (sparse.py:248)")
    else:
        c = f
    return np.ascontiguousarray(c, dtype=np.float64)


def chol_solve(factor, r: np.ndarray) -> np.ndarray:
    """``DenseFactor.solve`` for the Cholesky kind (sparse.py:225-230)."""
    kind = getattr(factor, "kind", "cholesky")
    if kind != "cholesky":
        raise NotImplementedError("the GPU hot path covers Cholesky factors only")
    c = _factor_array(factor)
    x = np.array(r, dtype=np.float64)
    if x.shape[0] != c.shape[0]:
        raise ValueError(f"dimension mismatch: factor is {c.shape[0]}, rhs has {x.shape[0]}")
    lib().oracle_chol_solve(c.shape[0], _p(c, _f64p), _p(x, _f64p))
    return x


class _Patches:
    def __init__(self, correction):
        idxs, facs = [], []
        for idx, factor in correction.regions:
            idxs.append(np.asarray(idx, dtype=np.int64))
            facs.append(_factor_array(factor))
        self.n_global = int(correction.n_global)
        self.ptr = np.zeros(len(idxs) + 1, dtype=np.int64)
        np.cumsum([len(i) for i in idxs], out=self.ptr[1:])
        self.idx = np.concatenate(idxs) if idxs else np.empty(0, dtype=np.int64)
        self.foff = np.zeros(len(facs) + 1, dtype=np.int64)
        np.cumsum([f.size for f in facs], out=self.foff[1:])
        self.factors = (np.concatenate([f.ravel() for f in facs]) if facs
                        else np.empty(0))


_pcache = {}


def _patches(correction) -> _Patches:
    hit = _pcache.get(id(correction))
    if hit is None or hit[0] is not correction:
        hit = (correction, _Patches(correction))
        _pcache[id(correction)] = hit
    return hit[1]


def apply_local_correction(correction, r: np.ndarray) -> np.ndarray:
    """smoothers.py:203-211: per-region exact solves, zero elsewhere."""
    r = np.asarray(r, dtype=np.float64)
    if r.shape != (correction.n_global,):
        raise ValueError(f"residual length {r.shape} does not match {correction.n_global}")
    pt = _patches(correction)
    out = np.zeros_like(r)
    x = np.ascontiguousarray(r[pt.idx])
    lib().oracle_patch_solves(len(pt.ptr) - 1, _p(pt.ptr, _i64p), _p(pt.foff, _i64p),
                              _p(pt.factors, _f64p), _p(x, _f64p))
    out[pt.idx] = x
    return out


def _local_residual_correction(a, b, u, correction) -> np.ndarray:
    """``apply_local_correction(correction, b - s @ u)`` evaluated on patch rows only.

    Off-patch residual entries never reach the output (smoothers.py:209-210), so
    computing only patch rows gives identical values.
    """
    pt = _patches(correction)
    rp = b[pt.idx] - spmv_rows(a, pt.idx, u)
    lib().oracle_patch_solves(len(pt.ptr) - 1, _p(pt.ptr, _i64p), _p(pt.foff, _i64p),
                              _p(pt.factors, _f64p), _p(rp, _f64p))
    out = np.zeros(len(u))
    out[pt.idx] = rp
    return out


# --------------------------------------------------------------------------
# smoothers (smoothers.py:99-136, 252-267)

class ZeroDiagonalError(ValueError):
    def __init__(self, row: int):
        super().__init__(f"zero diagonal entry in row {row}")
        self.row = row


def chebyshev_smooth(a, b: np.ndarray, u: np.ndarray, sweeps: int, cfg) -> np.ndarray:
    """smoothers.py:99-136, same expression order; updates ``u`` in place."""
    if cfg.lambda_max is None or cfg.lambda_max <= 0.0:
        raise ValueError("chebyshev_smooth requires a positive cfg.lambda_max")
    lam_max = cfg.lambda_max
    lam_min = cfg.lambda_min_fraction * lam_max
    diag = diagonal(a)
    zero = np.nonzero(diag == 0.0)[0]
    if len(zero):
        raise ZeroDiagonalError(int(zero[0]))
    inv_diag = 1.0 / diag

    theta = 0.5 * (lam_max + lam_min)
    delta = 0.5 * (lam_max - lam_min)
    if delta == 0.0:
        for _ in range(sweeps):
            u += inv_diag * (b - spmv(a, u)) / theta
        return u

    sigma = theta / delta
    rho = 1.0 / sigma
    d = inv_diag * (b - spmv(a, u)) / theta
    u += d
    for _ in range(sweeps - 1):
        rho_next = 1.0 / (2.0 * sigma - rho)
        z = inv_diag * (b - spmv(a, u))
        d = rho_next * rho * d + (2.0 * rho_next / delta) * z
        u += d
        rho = rho_next
    return u


def _cheb_cfg(cfg):
    """Map a ``kind='jacobi'`` config onto the reference's delta==0 branch
    (smoothers.py:120-124): lambda_max = 1/omega, fraction 1."""
    if getattr(cfg, "kind", "chebyshev") == "jacobi":
        class _C:
            pass
        c = _C()
        c.lambda_max = 1.0 / cfg.omega
        c.lambda_min_fraction = 1.0
        return c
    return cfg


def global_smooth(a, b, u, cfg) -> np.ndarray:
    if cfg.kind == "sgs":
        raise NotImplementedError("SGS is outside the GPU hot path (SURVEY.md section 2)")
    return chebyshev_smooth(a, b, u, cfg.sweeps, _cheb_cfg(cfg))


def combined_smooth(a, b, u, correction, cfg) -> np.ndarray:
    """smoothers.py:252-267 (sandwich); in place."""
    active = correction is not None and len(correction.regions) > 0
    if active:
        u += _local_residual_correction(a, b, u, correction)
    global_smooth(a, b, u, cfg)
    if active:
        u += _local_residual_correction(a, b, u, correction)
    return u


# --------------------------------------------------------------------------
# multigrid (mg.py:127-184)

def vcycle(h, b: np.ndarray, u: np.ndarray) -> np.ndarray:
    """mg.py:127-151; updates ``u`` in place."""
    n_levels = len(h.levels)
    b_levels: List[np.ndarray] = [np.asarray(b, dtype=np.float64)]
    u_levels: List[np.ndarray] = [u]
    for l in range(n_levels - 1):
        level = h.levels[l]
        combined_smooth(level.a, b_levels[l], u_levels[l], level.local_correction,
                        level.smoother)
        residual = b_levels[l] - spmv(level.a, u_levels[l])
        b_levels.append(spmv_transpose(level.prolongation.matrix, residual))
        u_levels.append(np.zeros(h.levels[l + 1].a.nrows))
    u_levels[-1][:] = chol_solve(h.coarse_factor, b_levels[-1])
    for l in range(n_levels - 2, -1, -1):
        level = h.levels[l]
        u_levels[l] += spmv(level.prolongation.matrix, u_levels[l + 1])
        combined_smooth(level.a, b_levels[l], u_levels[l], level.local_correction,
                        level.smoother)
    return u


def norm(x: np.ndarray) -> float:
    return float(np.sqrt(lib().oracle_dot(len(x), _p(np.ascontiguousarray(x), _f64p),
                                          _p(np.ascontiguousarray(x), _f64p))))


def solve_stationary(h, b, u0, rtol: float = 1e-10,
                     max_cycles: int = 100) -> Tuple[np.ndarray, List[float]]:
    """mg.py:154-175."""
    a = h.levels[0].a
    u = np.array(u0, dtype=np.float64)
    residual = norm(b - spmv(a, u))
    norm_b = norm(np.asarray(b, dtype=np.float64))
    denom = norm_b if norm_b > 0 else residual
    if denom == 0.0:
        return u, [0.0]
    history = [float(residual / denom)]
    for _ in range(max_cycles):
        if history[-1] <= rtol:
            break
        vcycle(h, b, u)
        history.append(float(norm(b - spmv(a, u)) / denom))
    return u, history


def as_preconditioner(h) -> Callable[[np.ndarray], np.ndarray]:
    """mg.py:178-184."""
    def apply(r):
        z = np.zeros_like(r)
        vcycle(h, r, z)
        return z
    return apply


class IndefiniteOperatorError(RuntimeError):
    def __init__(self, iteration: int, curvature: float):
        super().__init__(f"non-positive curvature p'Ap = {curvature:.6e} at CG iteration "
                         f"{iteration}; operator is not positive definite")
        self.iteration = iteration
        self.curvature = curvature


def cg(a, b, precond=None, rtol: float = 1e-10, maxit: int = 1000,
       x0: Optional[np.ndarray] = None):
    """sparse.py:168-211 with ``a`` a CSR matrix and ``precond`` a callable."""
    matvec = lambda v: spmv(a, v)
    apply_m = precond if precond is not None else (lambda v: v)
    dot = lambda p, q: float(lib().oracle_dot(len(p), _p(np.ascontiguousarray(p), _f64p),
                                              _p(np.ascontiguousarray(q), _f64p)))
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    r = b - matvec(x)
    norm_b = norm(b)
    denom = norm_b if norm_b > 0 else norm(r)
    if denom == 0.0:
        return x, [0.0]
    history = [float(norm(r) / denom)]
    if history[-1] <= rtol:
        return x, history
    z = apply_m(r)
    d = z.copy()
    rz = dot(r, z)
    for k in range(maxit):
        q = matvec(d)
        curvature = dot(d, q)
        if curvature <= 0.0:
            raise IndefiniteOperatorError(k, curvature)
        alpha = rz / curvature
        x += alpha * d
        r -= alpha * q
        history.append(float(norm(r) / denom))
        if history[-1] <= rtol:
            break
        z = apply_m(r)
        rz_new = dot(r, z)
        d = z + (rz_new / rz) * d
        rz = rz_new
    return x, history
