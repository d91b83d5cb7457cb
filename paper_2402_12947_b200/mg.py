"""Multigrid hierarchy and V-cycle solvers behind the reference's ``simplexmg.mg`` API.

Mirrors ``pkg/src/simplexmg/mg.py`` (paths relative to
/root/reference/pkg/src/simplexmg): ``Level`` / ``Hierarchy`` (:30-69),
``build_hierarchy`` (:72-124, setup on the host), ``vcycle`` (:127-151),
``solve_stationary`` (:154-175) and ``as_preconditioner`` (:178-184).

The solvers run entirely on the GPU through the C-ABI's device hierarchy
(``smg_hierarchy``): every level's operator, CSR(P^T) restriction, packed
patch factors and the dense coarse inverse live in HBM, and one V-cycle is a
single CUDA-graph launch.  ``DeviceHierarchy.from_reference(h)`` accepts the
reference's own ``Hierarchy`` object (duck-typed), so a reference user swaps
``simplexmg.mg.vcycle`` for ``paper_2402_12947_b200.mg.vcycle`` unchanged.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass, field, replace
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np
import scipy.linalg

from . import _lib
from . import device as _dev
from .sparse import CsrMatrix, DenseFactor, dense_factor
from .smoothers import (KIND_CODE, LocalCorrection, SmootherConfig, ZeroDiagonalError,
                        combined_smooth)

_f64p = ctypes.POINTER(ctypes.c_double)


@dataclass(frozen=True, eq=False)
class Prolongation:
    """Interpolation matrix from a coarse dof space into a finer one (transfer.py:104-114)."""

    matrix: CsrMatrix
    fine_level: Optional[int] = None
    coarse_level: Optional[int] = None

    @property
    def shape(self) -> tuple:
        return self.matrix.shape


@dataclass(eq=False)
class Level:
    """One grid level (mg.py:30-48)."""

    index: int
    mesh: object
    dofmap: object
    a: CsrMatrix
    prolongation: Optional[Prolongation]
    smoother: SmootherConfig
    regions: object
    local_correction: Optional[LocalCorrection]
    sgs: object = None
    lambda_max: Optional[float] = None
    lambda_max_adjusted: Optional[float] = None

    def smooth(self, b, u):
        return combined_smooth(self.a, b, u, self.local_correction, self.smoother, self.sgs)


@dataclass(eq=False)
class Hierarchy:
    """Levels fine to coarse plus the factored coarsest operator (mg.py:51-69)."""

    levels: List[Level]
    coarse_factor: DenseFactor
    system: object = None
    coarse_refine: bool = False

    @property
    def n_levels(self) -> int:
        return len(self.levels)

    @property
    def fine(self) -> Level:
        return self.levels[0]

    @property
    def rhs(self) -> np.ndarray:
        return self.system.b

    def device(self) -> "DeviceHierarchy":
        return _device_for(self)


def coarse_inverse(coarse_factor, device: Optional[bool] = None) -> np.ndarray:
    """Dense A_L^{-1} from the reference's Cholesky factor (mg.py:123) as
    LAPACK dpotri forms it (setup).  ``coarse_factor.factor = (c, lower)``.
    ``device`` (default: whenever a CUDA device exists): dpotri on the GPU
    (``smg_cholesky_inverse``, hand-written blocked dtrtri + dlauum) from the
    same factor."""
    f = getattr(coarse_factor, "factor", coarse_factor)
    kind = getattr(coarse_factor, "kind", "cholesky")
    if kind != "cholesky":
        raise NotImplementedError("coarse operator is not SPD (LU fallback): not on the GPU hot path")
    c, lower = f
    c = np.asarray(c, dtype=np.float64)
    if device is None:
        device = bool(_dev.torch().cuda.is_available())
    if device and c.size:
        lib = _lib.load()
        lo = np.ascontiguousarray(np.tril(c) if lower else np.triu(c).T)
        inv = np.empty_like(lo)
        _lib.check(lib.smg_cholesky_inverse(lo.shape[0], lo.ctypes.data_as(_f64p),
                                            inv.ctypes.data_as(_f64p), _dev.stream_handle()))
        return inv
    lo = np.asfortranarray(np.tril(c) if lower else np.triu(c).T)
    inv, info = scipy.linalg.lapack.dpotri(lo, lower=1)
    if info != 0:
        raise RuntimeError(f"dpotri failed with info={info}")
    tri = np.tril(inv)
    full = tri + tri.T
    full[np.diag_indices_from(full)] = np.diag(tri)
    return np.ascontiguousarray(full)


class DeviceHierarchy:
    """Device-resident hierarchy (smg_hierarchy): the object the solvers run on."""

    def __init__(self, levels, coarse_factor, coarse_refine: bool = False, use_graphs: bool = True,
                 coarse_inv: Optional[np.ndarray] = None):
        _dev.require_cuda()
        lib = _lib.load()
        nl = len(levels)
        if nl < 2:
            raise ValueError(f"a hierarchy needs at least 2 meshes, got {nl}")
        self.ops, self.prols, self.corrs = [], [], []
        kinds, sweeps, lmax, frac = [], [], [], []
        for l, lv in enumerate(levels):
            op = _dev.device_operator(lv.a)
            self.ops.append(op)
            if l < nl - 1:
                self.prols.append(_dev.device_operator(lv.prolongation.matrix, with_transpose=True))
                lc = lv.local_correction
                self.corrs.append(_dev.device_correction(lv.a, lc)
                                  if lc is not None and len(lc.regions) > 0 else None)
                cfg = SmootherConfig.from_any(lv.smoother)
                if cfg.kind == "sgs":
                    raise NotImplementedError("symmetric Gauss-Seidel is outside the GPU hot path")
                lm, fr = cfg.chebyshev_parameters()
                if lm is None or lm <= 0:
                    raise ValueError("chebyshev_smooth requires a positive cfg.lambda_max")
                if op.first_zero_diag >= 0:
                    raise ZeroDiagonalError(int(op.first_zero_diag))
                kinds.append(KIND_CODE[cfg.kind])
                sweeps.append(int(cfg.sweeps))
                lmax.append(float(lm))
                frac.append(float(fr))
            else:
                self.prols.append(None)
                self.corrs.append(None)
                kinds.append(0)
                sweeps.append(1)
                lmax.append(1.0)
                frac.append(0.1)
        self.n = [op.nrows for op in self.ops]
        inv = coarse_inverse(coarse_factor) if coarse_inv is None else coarse_inv
        n_c = self.n[-1]
        if inv.shape != (n_c, n_c):
            raise ValueError("coarse factor does not match the coarsest operator")
        self.coarse_inv = np.ascontiguousarray(inv)
        VP = ctypes.c_void_p * nl
        a_arr = VP(*[op.handle.value for op in self.ops])
        p_arr = VP(*[(p.handle.value if p is not None else None) for p in self.prols])
        c_arr = VP(*[(c.handle.value if c is not None else None) for c in self.corrs])
        IA = ctypes.c_int * nl
        DA = ctypes.c_double * nl
        h = ctypes.c_void_p()
        _lib.check(lib.smg_hierarchy_create(
            nl, ctypes.cast(a_arr, ctypes.POINTER(ctypes.c_void_p)),
            ctypes.cast(p_arr, ctypes.POINTER(ctypes.c_void_p)),
            ctypes.cast(c_arr, ctypes.POINTER(ctypes.c_void_p)),
            IA(*kinds), IA(*sweeps), DA(*lmax), DA(*frac), n_c,
            self.coarse_inv.ctypes.data_as(_f64p), 1 if coarse_refine else 0, ctypes.byref(h)))
        self.handle = h
        self._finalizer = weakref.finalize(self, lib.smg_hierarchy_destroy, h)
        self.set_graphs(use_graphs)

    @classmethod
    def from_reference(cls, h, coarse_refine: bool = False, use_graphs: bool = True):
        """Upload a reference ``simplexmg.mg.Hierarchy`` (or this package's)."""
        return cls(h.levels, h.coarse_factor, coarse_refine=coarse_refine, use_graphs=use_graphs)

    def set_graphs(self, enable: bool) -> None:
        _lib.check(_lib.load().smg_hierarchy_set_graphs(self.handle, 1 if enable else 0))

    def set_option(self, option: int, value: int) -> None:
        _lib.check(_lib.load().smg_hierarchy_set_option(self.handle, int(option), int(value)))

    def launches_per_vcycle(self) -> int:
        n = ctypes.c_int64()
        _lib.check(_lib.load().smg_hierarchy_launches_per_vcycle(self.handle, ctypes.byref(n)))
        return int(n.value)

    @property
    def n_levels(self) -> int:
        return len(self.ops)

    # -- solvers --------------------------------------------------------------
    def vcycle(self, b, u):
        n0 = self.n[0]
        lib = _lib.load()
        t = _dev.torch()
        if isinstance(u, t.Tensor):
            bt, _ = _dev.as_device_vector(b, n0, "b")
            ut, _ = _dev.as_device_vector(u, n0, "u")
            _lib.check(lib.smg_vcycle(self.handle, _dev.ptr(bt), _dev.ptr(ut),
                                      _dev.stream_handle()))
            return u
        bh = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
        if bh.shape != (n0,) or np.shape(u) != (n0,):
            raise ValueError(f"dimension mismatch: fine level has {n0} dofs")
        if not (isinstance(u, np.ndarray) and u.dtype == np.float64 and u.flags.c_contiguous):
            raise ValueError("u must be a contiguous float64 numpy array (updated in place)")
        _lib.check(lib.smg_vcycle_host(self.handle, bh.ctypes.data_as(_f64p),
                                       u.ctypes.data_as(_f64p), _dev.stream_handle()))
        return u

    def vcycles_host(self, bs, us):
        """One V-cycle on each independent host pair (bs[i], us[i]), us[i] in
        place, with the host<->device copies of neighbouring pairs overlapping
        each V-cycle (smg_vcycle_host_many; pinned arrays give the overlap)."""
        n0 = self.n[0]
        if len(bs) != len(us):
            raise ValueError("dimension mismatch: bs and us differ in length")
        for b, u in zip(bs, us):
            for name, a in (("b", b), ("u", u)):
                if not (isinstance(a, np.ndarray) and a.dtype == np.float64
                        and a.flags.c_contiguous and a.shape == (n0,)):
                    raise ValueError(f"{name} must be a contiguous float64 array of "
                                     f"{n0} dofs (dimension mismatch)")
        cnt = len(bs)
        bp = (ctypes.c_void_p * max(cnt, 1))(*[b.ctypes.data for b in bs])
        up = (ctypes.c_void_p * max(cnt, 1))(*[u.ctypes.data for u in us])
        _lib.check(_lib.load().smg_vcycle_host_many(self.handle, cnt, bp, up,
                                                    _dev.stream_handle()))
        return us

    def solve_stationary(self, b, u0, rtol: float = 1e-10, max_cycles: int = 100):
        n0 = self.n[0]
        t = _dev.torch()
        bt, host = _dev.as_device_vector(b, n0, "b")
        u0t, _ = _dev.as_device_vector(u0, n0, "u0")
        u = u0t.clone()
        hist = np.zeros(max_cycles + 2)
        nh = ctypes.c_int()
        _lib.check(_lib.load().smg_solve_stationary(
            self.handle, _dev.ptr(bt), _dev.ptr(u), float(rtol), int(max_cycles),
            hist.ctypes.data_as(_f64p), ctypes.byref(nh), _dev.stream_handle()))
        history = [float(v) for v in hist[:nh.value]]
        if host is not None or not isinstance(u0, t.Tensor):
            return u.cpu().numpy(), history
        return u, history

    def as_preconditioner(self) -> Callable:
        return as_preconditioner(self)

    def coarse_solve(self, b_c):
        """x_c = A_L^-1 b_c as the V-cycle applies it (mg.py:145;
        smg_coarse_solve).  numpy in -> numpy out; CUDA tensor -> tensor."""
        t = _dev.torch()
        bt, host = _dev.as_device_vector(b_c, self.n[-1], "b_c")
        x = t.empty_like(bt)
        _lib.check(_lib.load().smg_coarse_solve(self.handle, _dev.ptr(bt), _dev.ptr(x),
                                                _dev.stream_handle()))
        return x.cpu().numpy() if host is not None and not isinstance(b_c, t.Tensor) else x


def _signature(h) -> tuple:
    sig = []
    for lv in h.levels:
        cfg = lv.smoother
        sig.append((id(lv.a), id(lv.prolongation) if lv.prolongation is not None else None,
                    id(lv.local_correction), cfg.kind, cfg.sweeps, cfg.lambda_max,
                    cfg.lambda_min_fraction, getattr(cfg, "omega", None)))
    sig.append(id(h.coarse_factor))
    sig.append(bool(getattr(h, "coarse_refine", False)))
    return tuple(sig)


_dev_cache = {}


def _device_for(h) -> DeviceHierarchy:
    key = id(h)
    sig = _signature(h)
    hit = _dev_cache.get(key)
    if hit is not None and hit[0]() is h and hit[1] == sig:
        return hit[2]
    dh = DeviceHierarchy(h.levels, h.coarse_factor,
                         coarse_refine=bool(getattr(h, "coarse_refine", False)))
    try:
        ref = weakref.ref(h, lambda _r, k=key: _dev_cache.pop(k, None))
    except TypeError:
        ref = (lambda o=h: o)
    _dev_cache[key] = (ref, sig, dh)
    return dh


def _as_device_hierarchy(obj) -> Optional[DeviceHierarchy]:
    if isinstance(obj, DeviceHierarchy):
        return obj
    dh = getattr(obj, "_smg_device_hierarchy", None)
    if dh is not None:
        return dh
    if hasattr(obj, "levels") and hasattr(obj, "coarse_factor"):
        return _device_for(obj)
    return None


def vcycle(h, b, u):
    """One V-cycle, ``u`` updated in place (mg.py:127-151)."""
    return _as_device_hierarchy(h).vcycle(b, u)


def solve_stationary(h, b, u0, rtol: float = 1e-10,
                     max_cycles: int = 100) -> Tuple[np.ndarray, List[float]]:
    """Repeat V-cycles until the relative residual drops below rtol (mg.py:154-175)."""
    return _as_device_hierarchy(h).solve_stationary(b, u0, rtol, max_cycles)


def as_preconditioner(h) -> Callable:
    """r -> vcycle(0; r) (mg.py:178-184).  The callable carries its device
    hierarchy so :func:`paper_2402_12947_b200.sparse.cg` runs it on-device."""
    dh = _as_device_hierarchy(h)

    def apply(r):
        t = _dev.torch()
        if isinstance(r, t.Tensor):
            z = t.zeros_like(r)
        else:
            z = np.zeros_like(np.asarray(r, dtype=np.float64))
        dh.vcycle(r, z)
        return z

    apply._smg_device_hierarchy = dh
    return apply


# ---------------------------------------------------------------------------
# setup (host): mg.py:72-124 restated over this package's vectorised builders

@dataclass(frozen=True)
class ProblemSpec:
    """The reference's problem data (fem.py:230-262), restricted to what the
    GPU setup assembles: Poisson with homogeneous Dirichlet data on every box
    face.  ``source``: f(x) for one point (as the reference evaluates it,
    fem.py:288-300) or, with ``vectorized_source=True``, f(points) for an
    (m, dim) array."""

    kind: str = "poisson"
    source: Optional[Callable] = None
    dirichlet: tuple = ()
    neumann: tuple = ()
    material: Optional[dict] = None
    vectorized_source: bool = False


def _vector_source(problem):
    """A vectorised (m, dim) -> (m,) source from a reference-style ProblemSpec."""
    f = getattr(problem, "source", None)
    if f is None:
        return None
    if getattr(problem, "vectorized_source", False):
        return f
    return lambda pts: np.fromiter((float(f(p)) for p in pts), dtype=np.float64, count=len(pts))


def _check_problem(problem, dim: int) -> None:
    kind = getattr(problem, "kind", None)
    if kind != "poisson":
        raise NotImplementedError(f"problem kind {kind!r}: the GPU setup assembles Poisson only "
                                  "(elasticity is outside the hot path, SURVEY.md section 2)")
    if tuple(getattr(problem, "neumann", ()) or ()):
        raise NotImplementedError("Neumann data is outside the GPU setup (homogeneous Dirichlet "
                                  "on every box face)")
    markers = sorted(int(m) for m, _ in getattr(problem, "dirichlet", ()))
    if markers != list(range(1, 2 * dim + 1)):
        raise NotImplementedError("the GPU setup eliminates Dirichlet conditions on every box face "
                                  f"(markers 1..{2 * dim}); got {markers}")
    probe = np.full(dim, 0.5)
    for _, fn in problem.dirichlet:
        val = np.asarray(fn(probe), dtype=np.float64)
        if np.any(val != 0.0):
            raise NotImplementedError("only homogeneous Dirichlet data is supported")


def _own_mesh(m):
    from .mesh import SimplexMesh
    if isinstance(m, SimplexMesh):
        return m
    return SimplexMesh(int(m.dim), np.asarray(m.vertices, dtype=np.float64),
                       np.asarray(m.cells, dtype=np.int64), np.asarray(m.boundary_facets, dtype=np.int64),
                       np.asarray(m.facet_markers, dtype=np.int64))


def build_hierarchy(meshes: Sequence, problem, smoother: SmootherConfig,
                    use_local_correction: bool, quality_threshold: float = 0.1,
                    element_degree: int = 1, *, region_layers: int = 1,
                    lambda_tol: float = 1e-8, coarse_refine: bool = False,
                    device_setup: Optional[bool] = None,
                    device_assembly=None) -> Hierarchy:
    """``build_hierarchy(meshes, problem, smoother, use_local_correction,
    quality_threshold=0.1, element_degree=1)`` as the reference (mg.py:72-124);
    meshes fine to coarse (reference ``SimplexMesh`` objects are accepted),
    ``problem`` a Poisson ``ProblemSpec`` (the reference's or this package's)
    with homogeneous Dirichlet data on every box face.

    ``device_setup``: prolongations (point location, ``smg_prolongation_build``),
    Galerkin products (``smg_galerkin``), patch Cholesky factors, the coarse
    factor and Lanczos on levels >= 200k rows run on the GPU (default:
    whenever a CUDA device exists).  The fine operator's element matrices
    are always formed on the host with the reference's own arithmetic (numpy
    einsum / LAPACK det and inv); with device setup the duplicate summation
    (in scipy's exact order) and the Dirichlet elimination run on the GPU
    (``smg_assemble_elements``), so A_0 and therefore every Galerkin level
    are bit-identical to the reference's construction either way.
    ``device_assembly="kernel"`` forms the element matrices on the GPU too
    (``smg_assemble_poisson``: same pattern, values within ~1e-13, so
    exact-zero Galerkin sums can differ -- a setup-time shortcut only).
    Host-only setup (no GPU, e.g. the CPU test suite) uses the reference's
    own scipy products."""
    if isinstance(problem, SmootherConfig) or hasattr(problem, "sweeps"):
        raise TypeError("build_hierarchy(meshes, problem, smoother, use_local_correction, ...): "
                        "the second argument is the ProblemSpec (mg.py:72-75)")
    meshes = [_own_mesh(m) for m in meshes]
    if len(meshes) < 2:
        raise ValueError(f"a hierarchy needs at least 2 meshes, got {len(meshes)}")
    if len({m.dim for m in meshes}) != 1:
        raise ValueError("all meshes must share the same dimension")
    _check_problem(problem, meshes[0].dim)
    source = _vector_source(problem)
    smoother = SmootherConfig.from_any(smoother)
    from .fem import assemble_poisson, build_dofmap
    from .mesh import identify_regions
    from .smoothers import (adjusted_lambda_max, build_local_correction, dofs_for_regions,
                            jacobi_lambda_max)
    from .transfer import build_prolongation, coarsen_system
    if device_setup is None:
        from .device import torch
        device_setup = bool(torch().cuda.is_available())
    import time
    times = {"dofmap_s": 0.0, "assembly_s": 0.0, "prolongation_s": 0.0, "galerkin_s": 0.0,
             "regions_s": 0.0, "local_factor_s": 0.0, "lambda_s": 0.0, "coarse_factor_s": 0.0}
    t = time.perf_counter()
    dofmaps = [build_dofmap(m, element_degree) for m in meshes]
    times["dofmap_s"] += time.perf_counter() - t
    t = time.perf_counter()
    if device_assembly is None:
        device_assembly = bool(device_setup)
    system = assemble_poisson(meshes[0], dofmaps[0], source,
                              device=device_assembly if device_setup else False)
    times["assembly_s"] += time.perf_counter() - t
    operators = [system.a]
    prolongations = []
    for l in range(len(meshes) - 1):
        t = time.perf_counter()
        p = build_prolongation(dofmaps[l], meshes[l + 1], dofmaps[l + 1], device=device_setup)
        prolongations.append(Prolongation(p, l, l + 1))
        times["prolongation_s"] += time.perf_counter() - t
        t = time.perf_counter()
        operators.append(coarsen_system(operators[l], p, device=device_setup))
        times["galerkin_s"] += time.perf_counter() - t
    levels = []
    for l, (mesh, dofmap, a) in enumerate(zip(meshes, dofmaps, operators)):
        t = time.perf_counter()
        regions = identify_regions(mesh, quality_threshold, layers=region_layers)
        dof_sets = dofs_for_regions(dofmap, mesh, regions)
        times["regions_s"] += time.perf_counter() - t
        correction = None
        if use_local_correction and dof_sets:
            t = time.perf_counter()
            correction = build_local_correction(a, dof_sets, device=device_setup)
            times["local_factor_s"] += time.perf_counter() - t
        lam = lam_adj = None
        cfg = smoother
        if smoother.kind == "chebyshev":
            t = time.perf_counter()
            lam = jacobi_lambda_max(a, lambda_tol, device_setup)
            lam_adj = (adjusted_lambda_max(a, dof_sets, lambda_tol, device_setup)
                       if dof_sets else lam)
            cfg = replace(smoother, lambda_max=lam_adj if smoother.adjusted else lam)
            times["lambda_s"] += time.perf_counter() - t
        prol = prolongations[l] if l < len(prolongations) else None
        levels.append(Level(l, mesh, dofmap, a, prol, cfg, regions, correction, None, lam, lam_adj))
    t = time.perf_counter()
    coarse = dense_factor(operators[-1].to_dense(), device=device_setup)
    times["coarse_factor_s"] += time.perf_counter() - t
    h = Hierarchy(levels, coarse, system, coarse_refine)
    h.setup_times = dict(times, galerkin_device=bool(device_setup),
                         assembly_device=str(device_assembly) if device_setup else "host")
    return h
