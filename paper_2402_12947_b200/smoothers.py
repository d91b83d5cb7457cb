"""GPU smoothers behind the reference's ``simplexmg.smoothers`` API.

Mirrors ``pkg/src/simplexmg/smoothers.py`` (paths relative to
/root/reference/pkg/src/simplexmg):

* ``SmootherConfig`` (:33-59) -- adds ``kind="jacobi"`` with ``omega``, which
  maps onto the reference's collapsed-interval branch (:120-124) with
  ``lambda_max = 1/omega`` and ``lambda_min_fraction = 1`` (SURVEY.md
  finding 3), i.e. exactly ``u += D^-1 (b - A u) / theta``.
* ``chebyshev_smooth`` (:99-136), ``apply_local_correction`` (:203-211) and
  ``combined_smooth`` (:252-267) run on the GPU (bit-identical SpMV-based
  steps; Cholesky patch solves to ~1e-15).  Numpy inputs are copied in and
  the in-place update is written back into the caller's array; CUDA float64
  tensors are updated in place on the device.
* ``LocalCorrection`` / ``build_local_correction`` (:139-200) and
  ``dofs_for_regions`` (:161-173) are setup (host, scipy Cholesky).
* ``sgs_sweep`` is outside the GPU hot path and raises
  NotImplementedError instead of silently running on the CPU.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from . import device as _dev
from .sparse import (DEVICE_LANCZOS_MIN_ROWS, CsrMatrix, DenseFactor, NotPositiveDefiniteError,
                     dense_factor, device_matvec, estimate_lambda_max)


class ZeroDiagonalError(ValueError):
    def __init__(self, row: int):
        super().__init__(f"zero diagonal entry in row {row}")
        self.row = row


@dataclass
class SmootherConfig:
    """Global smoother selection (smoothers.py:33-59) plus ``jacobi``."""

    kind: str = "sgs"
    sweeps: int = 1
    lambda_max: Optional[float] = None
    lambda_min_fraction: float = 0.1
    adjusted: bool = False
    omega: Optional[float] = None

    def __post_init__(self):
        if self.kind not in ("sgs", "chebyshev", "jacobi"):
            raise ValueError(f"unknown smoother kind {self.kind!r}")
        if self.sweeps < 1:
            raise ValueError(f"sweeps must be at least 1, got {self.sweeps}")
        if not 0.0 < self.lambda_min_fraction <= 1.0:
            raise ValueError(f"lambda_min_fraction must lie in (0, 1], got {self.lambda_min_fraction}")
        if self.lambda_max is not None and self.lambda_max <= 0.0:
            raise ValueError(f"lambda_max must be positive, got {self.lambda_max}")
        if self.kind == "jacobi":
            if self.omega is None or not self.omega > 0.0:
                raise ValueError("jacobi smoother needs a positive omega")

    def chebyshev_parameters(self) -> Tuple[float, float]:
        """(lambda_max, lambda_min_fraction) as the reference arithmetic sees them."""
        if self.kind == "jacobi":
            return 1.0 / self.omega, 1.0
        return self.lambda_max, self.lambda_min_fraction

    @classmethod
    def from_any(cls, cfg) -> "SmootherConfig":
        if isinstance(cfg, cls):
            return cfg
        return cls(kind=cfg.kind, sweeps=cfg.sweeps, lambda_max=cfg.lambda_max,
                   lambda_min_fraction=cfg.lambda_min_fraction,
                   adjusted=getattr(cfg, "adjusted", False), omega=getattr(cfg, "omega", None))


KIND_CODE = {"chebyshev": 0, "jacobi": 0, "sgs": 1}


@dataclass(frozen=True, eq=False)
class LocalCorrection:
    """Disjoint dof sets with Cholesky factors of their principal submatrices."""

    regions: Tuple[Tuple[np.ndarray, DenseFactor], ...]
    n_global: int

    @property
    def n_regions(self) -> int:
        return len(self.regions)

    @property
    def covered_dofs(self) -> np.ndarray:
        if not self.regions:
            return np.empty(0, dtype=np.int64)
        return np.concatenate([idx for idx, _ in self.regions])


def dofs_for_regions(dofmap, mesh, regions) -> List[np.ndarray]:
    """Dof sets of the cells of each region (smoothers.py:161-173; scalar fields)."""
    return [np.unique(dofmap.cell_nodes[np.asarray(r, dtype=np.int64)])
            for r in regions.omega_B_regions]


def build_local_correction(a, dof_sets: Sequence[np.ndarray],
                           device: Optional[bool] = None) -> LocalCorrection:
    """smoothers.py:176-200 (setup): factor each principal submatrix.

    ``device`` (default: whenever a CUDA device exists): every block is
    gathered and Cholesky-factored on the GPU in one batched launch
    (``smg_patch_factor``, one CTA per region); otherwise scipy cho_factor
    per block as the reference does.  Same validation order and errors."""
    a = CsrMatrix.from_any(a)
    if device is None:
        device = bool(_dev.torch().cuda.is_available())
    regions = []
    kept = []
    seen = np.zeros(a.nrows, dtype=bool)
    s = None if device else a.to_scipy()
    for k, dofs in enumerate(dof_sets):
        idx = np.unique(np.asarray(dofs, dtype=np.int64))
        if len(idx) == 0:
            continue
        if idx[0] < 0 or idx[-1] >= a.nrows:
            raise ValueError(f"region {k} has dof indices outside 0..{a.nrows - 1}")
        if np.any(seen[idx]):
            raise ValueError(f"region {k} overlaps a previous region's dofs")
        seen[idx] = True
        if device:
            kept.append((k, idx))
            continue
        sub = s[idx][:, idx].toarray()
        try:
            factor = dense_factor(sub, lu_fallback=False)
        except NotPositiveDefiniteError as err:
            raise NotPositiveDefiniteError(
                f"local block {k} ({len(idx)} dofs) is not SPD: {err}") from err
        regions.append((idx, factor))
    if device and kept:
        regions = _factor_blocks_device(a, kept)
    return LocalCorrection(tuple(regions), a.nrows)


def _factor_blocks_device(a, kept) -> list:
    import ctypes
    lib = _lib.load()
    op = _dev.device_operator(a)
    sizes = np.array([len(idx) for _, idx in kept], dtype=np.int64)
    roff = np.zeros(len(kept) + 1, dtype=np.int64)
    np.cumsum(sizes, out=roff[1:])
    dofs = np.ascontiguousarray(np.concatenate([idx for _, idx in kept]), dtype=np.int64)
    foff = np.zeros(len(kept) + 1, dtype=np.int64)
    np.cumsum(sizes * sizes, out=foff[1:])
    factors = np.empty(int(foff[-1]))
    bad_r, bad_minor = ctypes.c_int64(-1), ctypes.c_int64(0)
    i64p = ctypes.POINTER(ctypes.c_int64)
    rc = lib.smg_patch_factor(op.handle, len(kept), roff.ctypes.data_as(i64p),
                              dofs.ctypes.data_as(i64p),
                              factors.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                              ctypes.byref(bad_r), ctypes.byref(bad_minor), _dev.stream_handle())
    if rc == _lib.SMG_ERR_NOT_SPD:
        k, idx = kept[bad_r.value]
        raise NotPositiveDefiniteError(
            f"local block {k} ({len(idx)} dofs) is not SPD: Cholesky failed: "
            f"{bad_minor.value}-th leading minor not positive definite")
    if rc == _lib.SMG_ERR_INVALID and bad_r.value >= 0:
        raise ValueError("dense_factor expects a symmetric matrix")
    _lib.check(rc)
    out = []
    for r, (k, idx) in enumerate(kept):
        nd = len(idx)
        c = factors[foff[r]:foff[r + 1]].reshape(nd, nd)
        out.append((idx, DenseFactor("cholesky", (c, True), nd)))
    return out


def _check_diag(op) -> None:
    if op.first_zero_diag >= 0:
        raise ZeroDiagonalError(int(op.first_zero_diag))


def _raise_mapped(err: _lib.SmgError):
    if err.code == _lib.SMG_ERR_UNSUPPORTED:
        raise NotImplementedError(str(err)) from None
    if err.code in (_lib.SMG_ERR_INVALID, _lib.SMG_ERR_DIMENSION):
        raise ValueError(str(err)) from None
    raise err


def _write_back(u, ut, host):
    if host is not None:
        u[...] = ut.cpu().numpy()
    return u


def chebyshev_smooth(a, b, u, sweeps: int, cfg):
    """Degree-``sweeps`` Jacobi-preconditioned Chebyshev (smoothers.py:99-136), in place."""
    cfg = SmootherConfig.from_any(cfg)
    lam_max, frac = cfg.chebyshev_parameters()
    if lam_max is None or lam_max <= 0.0:
        raise ValueError("chebyshev_smooth requires a positive cfg.lambda_max")
    op = _dev.device_operator(a)
    _check_diag(op)
    bt, _ = _dev.as_device_vector(b, op.nrows, "b")
    ut, host = _dev.as_device_vector(u, op.nrows, "u")
    try:
        _lib.check(_lib.load().smg_chebyshev_smooth(op.handle, _dev.ptr(bt), _dev.ptr(ut),
                                                    int(sweeps), float(lam_max), float(frac),
                                                    None, _dev.stream_handle()))
    except _lib.SmgError as e:
        _raise_mapped(e)
    return _write_back(u, ut, host)


def sgs_sweep(*args, **kwargs):
    raise NotImplementedError("symmetric Gauss-Seidel is outside the GPU hot path "
                              "(SURVEY.md section 2); use the reference package for SGS")


def apply_local_correction(correction, r):
    """Sum of the per-region corrections, zero elsewhere (smoothers.py:203-211)."""
    n = int(correction.n_global)
    rt, host = _dev.as_device_vector(r, None, "r")
    if rt.shape != (n,):
        raise ValueError(f"residual length {tuple(rt.shape)} does not match {n}")
    dc = _corr_handle(correction, n)
    t = _dev.torch()
    out = t.empty(n, dtype=t.float64, device=rt.device)
    _lib.check(_lib.load().smg_apply_local_correction(dc.handle, _dev.ptr(rt), _dev.ptr(out),
                                                      _dev.stream_handle()))
    return out.cpu().numpy() if host is not None else out


_standalone = {}


def _corr_handle(correction, n):
    """A LocalCorrection needs an operator only for its residuals; for the
    standalone apply path an identity-sized dummy operator suffices."""
    key = id(correction)
    hit = _standalone.get(key)
    if hit is not None and hit[0] is correction:
        return hit[1]
    dummy = CsrMatrix.identity(n)
    dc = _dev.DeviceCorrection(_dev.DeviceOperator(dummy), correction)
    _standalone[key] = (correction, dc)
    return dc


def combined_smooth(a, b, u, correction, cfg, splitting=None):
    """Sandwich smoother S_c, global smoother, S_c (smoothers.py:252-267), in place."""
    cfg = SmootherConfig.from_any(cfg)
    if cfg.kind == "sgs":
        sgs_sweep()
    lam_max, frac = cfg.chebyshev_parameters()
    if lam_max is None or lam_max <= 0.0:
        raise ValueError("chebyshev_smooth requires a positive cfg.lambda_max")
    op = _dev.device_operator(a)
    _check_diag(op)
    bt, _ = _dev.as_device_vector(b, op.nrows, "b")
    ut, host = _dev.as_device_vector(u, op.nrows, "u")
    active = correction is not None and len(correction.regions) > 0
    dc = _dev.device_correction(a, correction) if active else None
    try:
        _lib.check(_lib.load().smg_combined_smooth(
            op.handle, _dev.ptr(bt), _dev.ptr(ut), dc.handle if dc else None,
            KIND_CODE[cfg.kind], int(cfg.sweeps), float(lam_max), float(frac), None,
            _dev.stream_handle()))
    except _lib.SmgError as e:
        _raise_mapped(e)
    return _write_back(u, ut, host)


def jacobi_lambda_max(a, tol: float = 1e-8, device: Optional[bool] = None) -> float:
    """Largest eigenvalue of D^-1 A (smoothers.py:214-222; setup).  ``device``
    (default: whenever a CUDA device exists) runs the Lanczos matvecs of
    operators with at least DEVICE_LANCZOS_MIN_ROWS rows on the GPU (bitwise
    equal SpMV, so the estimate is the host path's, which is the
    reference's)."""
    a = CsrMatrix.from_any(a)
    diag = a.diagonal()
    zero = np.nonzero(diag == 0.0)[0]
    if len(zero):
        raise ZeroDiagonalError(int(zero[0]))
    scale = 1.0 / np.sqrt(np.abs(diag))
    if device is None:
        device = bool(_dev.torch().cuda.is_available())
    if a.nrows >= DEVICE_LANCZOS_MIN_ROWS and device:
        return estimate_lambda_max(device_matvec(a, scale), a.nrows, tol)
    s = a.to_scipy()
    return estimate_lambda_max(lambda x: scale * (s @ (scale * x)), a.nrows, tol)


def adjusted_lambda_max(a, boundary_dof_sets: Sequence[np.ndarray], tol: float = 1e-8,
                        device: Optional[bool] = None) -> float:
    """smoothers.py:225-241 (setup)."""
    a = CsrMatrix.from_any(a)
    covered = np.zeros(a.nrows, dtype=bool)
    for dofs in boundary_dof_sets:
        covered[np.asarray(dofs, dtype=np.int64)] = True
    keep = np.nonzero(~covered)[0]
    if len(keep) == 0:
        raise ValueError("excluded dofs cover the whole operator; nothing remains")
    if len(keep) == a.nrows:
        return jacobi_lambda_max(a, tol, device)
    return jacobi_lambda_max(a.principal_submatrix(keep), tol, device)
