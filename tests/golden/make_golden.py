"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

    python tests/golden/make_golden.py            # needs /root/reference

Every output vector here comes from the reference's own functions
(`simplexmg` imported through refshim, unmodified), on seeded inputs:

* crit7_adj / crit7_ref -- the acceptance suite's criterion-7 experiments
  (pkg/tests/test_acceptance.py:226-242; config shape as :41-51): P2
  square, 4 levels (46/23/12/6), Chebyshev degree 2 (adjusted lambda), local
  correction; and the unperturbed "reference" case.  Stored: hierarchy,
  per-sweep Chebyshev vectors, sandwich smoother, V-cycles, stationary and
  CG residual histories / iteration counts.
* c1s, c2s, c3s -- BASELINE C1/C2/C3 constructions at reduced grids
  (paper_2402_12947_b200.configs .scaled): meshes from this repo's
  construction, everything else (assembly, transfer, Galerkin, regions,
  factors, lambda, solves) by the reference.  C1/C3 use the reference's
  damped-Jacobi branch (lambda_max = 1.5, fraction 1 => omega = 2/3,
  smoothers.py:120-124); C2 uses 2-layer regions computed harness-side and
  factored by the reference's build_local_correction.
* c4s -- BASELINE C4 construction (3D P2, flattened tets, Chebyshev
  degree 2) at grids 12/6/3/2 with two clusters: two 279-dof regions, past
  the shared-memory cap, so the streamed-factor patch path runs.
* c5p -- C5-style batched patch solves: dense SPD blocks of 64/200/512 dofs,
  cond 1e6, embedded in an otherwise-identity operator; reference
  apply_local_correction outputs.
* cpl_p1, cpl_p2, unc_p2 -- several local-correction regions on one level
  (SURVEY.md A4), every step by the reference: a 16x16 grid whose flattened
  vertices (the reference's _apply_clusters) sit 4 cells apart (two regions
  coupled through A; P1 and P2), or far apart (three uncoupled regions).

``python tests/golden/make_golden.py c4s cpl_p1`` regenerates only those.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from tests.golden import fixtures, refshim  # noqa: E402


def _ref():
    return refshim.import_reference()


def _common_goldens(sm, h, b, u0, d, prefix="g", cg_maxit=300, rtol=1e-10, max_cycles=300):
    mg, smo, sparse = sm.mg, sm.smoothers, sm.sparse
    lv = h.levels[0]
    n = lv.a.nrows
    rng = np.random.default_rng(11)
    ur = rng.standard_normal(n)
    d[prefix + "/u_rand"] = ur
    d[prefix + "/b"] = np.asarray(b, dtype=np.float64)
    d[prefix + "/u0"] = np.asarray(u0, dtype=np.float64)
    s = lv.a.to_scipy()
    d[prefix + "/spmv"] = s @ ur
    d[prefix + "/residual"] = b - s @ ur
    pm = lv.prolongation.matrix.to_scipy()
    d[prefix + "/restrict"] = pm.T @ ur
    uc = rng.standard_normal(pm.shape[1])
    d[prefix + "/uc"] = uc
    uf = ur.copy()
    uf += pm @ uc
    d[prefix + "/prolong_add"] = uf
    cfg = lv.smoother
    for k in range(1, cfg.sweeps + 1):
        d[prefix + f"/cheb{k}"] = smo.chebyshev_smooth(lv.a, b, ur.copy(), k, cfg)
    d[prefix + "/combined"] = smo.combined_smooth(lv.a, b, ur.copy(), lv.local_correction, cfg)
    if lv.local_correction is not None:
        r = b - s @ ur
        d[prefix + "/lc_apply"] = smo.apply_local_correction(lv.local_correction, r)
    v1 = mg.vcycle(h, b, ur.copy())
    d[prefix + "/vcycle1"] = v1.copy()
    d[prefix + "/vcycle2"] = mg.vcycle(h, b, v1.copy())
    d[prefix + "/vcycle_zero"] = mg.vcycle(h, b, np.zeros(n))
    u, hist = mg.solve_stationary(h, b, u0, rtol=rtol, max_cycles=max_cycles)
    d[prefix + "/stat_hist"] = np.asarray(hist)
    d[prefix + "/stat_u"] = u
    hits = [k for k, r in enumerate(hist) if r <= rtol]
    d[prefix + "/stat_iters"] = np.array(hits[0] if hits else -1)
    x, chist = sparse.cg(lv.a, b, precond=mg.as_preconditioner(h), rtol=rtol, maxit=cg_maxit)
    d[prefix + "/cg_hist"] = np.asarray(chist)
    d[prefix + "/cg_x"] = x
    hits = [k for k, r in enumerate(chist) if r <= rtol]
    d[prefix + "/cg_iters"] = np.array(hits[0] if hits else -1)
    # coarse solve golden
    nc = h.levels[-1].a.nrows
    bc = rng.standard_normal(nc)
    d[prefix + "/coarse_b"] = bc
    d[prefix + "/coarse_x"] = h.coarse_factor.solve(bc)
    return d


def _versions(d):
    import scipy
    d["meta/numpy"] = np.array(np.__version__)
    d["meta/scipy"] = np.array(scipy.__version__)


def crit7():
    sm = _ref()
    ex = sm.experiments

    def cfg(case, correction, smoother):
        return ex.ExperimentConfig(
            problem="poisson", dim=2, element_degree=2, case=case,
            levels=({"n": 46}, {"n": 23}, {"n": 12}, {"n": 6}),
            clusters=({"center": (0.3, 0.3), "gamma": 1e-4, "vertices": 1},),
            smoother=smoother, local_correction=correction, mode="stationary",
            rtol=1e-10, max_iterations=300, seed=0, boundary="y", source="cos-sin",
            initial_guess="zero")

    cheb = {"kind": "chebyshev", "sweeps": 2, "adjusted": False}
    cheb_adj = {"kind": "chebyshev", "sweeps": 2, "adjusted": True}
    out = {}
    for name, c in (("crit7_adj", cfg("A", True, cheb_adj)), ("crit7_ref", cfg("reference", False, cheb))):
        h = ex.build_experiment(c)
        u0 = ex._initial_guess(c, h)
        d = fixtures.hierarchy_arrays(h)
        _common_goldens(sm, h, h.rhs, u0, d)
        d["lambda_max"] = np.array([lv.lambda_max for lv in h.levels])
        d["lambda_max_adjusted"] = np.array([lv.lambda_max_adjusted for lv in h.levels])
        report = ex.run(c)
        d["run_iters"] = np.array(report.iterations_to_rtol)
        out[name] = (d, h, u0)
    # unadjusted count on the same (case A) hierarchy: only lambda changes
    d, h, u0 = out["crit7_adj"]
    report = ex.run(cfg("A", True, cheb))
    d["unadjusted_run_iters"] = np.array(report.iterations_to_rtol)
    from dataclasses import replace
    saved = [lv.smoother for lv in h.levels]
    for lv in h.levels:
        lv.smoother = replace(lv.smoother, lambda_max=lv.lambda_max)
    _, hist = sm.mg.solve_stationary(h, h.rhs, u0, 1e-10, 300)
    hits = [k for k, r in enumerate(hist) if r <= 1e-10]
    d["unadjusted_stat_hist"] = np.asarray(hist)
    d["unadjusted_stat_iters"] = np.array(hits[0])
    for lv, s in zip(h.levels, saved):
        lv.smoother = s
    for name, (d, _, _) in out.items():
        _versions(d)
        np.savez_compressed(fixtures.path(name), **d)
        print(name, "iters", int(d["g/stat_iters"]), "run", int(d["run_iters"]))


def _ref_meshes(sm, meshes):
    return [sm.mesh.SimplexMesh(m.dim, m.vertices, m.cells, m.boundary_facets, m.facet_markers)
            for m in meshes]


def baseline_small(name, wl, jacobi_theta=None, layers=1):
    sm = _ref()
    from paper_2402_12947_b200 import configs
    from paper_2402_12947_b200.mesh import identify_regions
    meshes = configs.build_meshes(wl)
    rmeshes = _ref_meshes(sm, meshes)
    dim = wl.dim
    zero = lambda x: 0.0
    source = (lambda x: 1.0) if wl.rhs == "source-one" else None
    problem = sm.fem.ProblemSpec("poisson", source=source,
                                 dirichlet=tuple((m, zero) for m in range(1, 2 * dim + 1)))
    kind_sweeps = wl.smoother.sweeps
    smoother = sm.smoothers.SmootherConfig("chebyshev", kind_sweeps)
    use_lc = layers == 1
    h = sm.mg.build_hierarchy(rmeshes, problem, smoother, use_lc, 0.1, wl.degree)
    if layers != 1:
        for lv, mesh in zip(h.levels, meshes):
            regs = identify_regions(mesh, 0.1, layers=layers)
            sets = [np.unique(lv.dofmap.cell_nodes[r]) for r in regs.omega_B_regions]
            if sets:
                lv.local_correction = sm.smoothers.build_local_correction(lv.a, sets)
    if jacobi_theta is not None:
        for lv in h.levels:
            lv.smoother = sm.smoothers.SmootherConfig("chebyshev", kind_sweeps,
                                                      lambda_max=jacobi_theta,
                                                      lambda_min_fraction=1.0)
    n0 = h.levels[0].a.nrows
    if wl.rhs == "random":
        b = np.random.default_rng([wl.seed, 99]).standard_normal(n0)
        b[h.system.dirichlet_dofs] = 0.0
    else:
        b = np.array(h.system.b)
    u0 = np.zeros(n0)
    d = fixtures.hierarchy_arrays(h)
    _common_goldens(sm, h, b, u0, d)
    d["meta/grids"] = np.array(wl.grids)
    _versions(d)
    np.savez_compressed(fixtures.path(name), **d)
    print(name, [lv.a.nrows for lv in h.levels], "stat iters", int(d["g/stat_iters"]),
          "cg iters", int(d["g/cg_iters"]),
          "regions", [0 if lv.local_correction is None else lv.local_correction.n_regions
                      for lv in h.levels])


def c5_patches():
    sm = _ref()
    rng = np.random.default_rng(2402)
    sizes = [64, 200, 512]
    n = 1600
    perm = rng.permutation(n)
    sets, start = [], 0
    rows, cols, vals = [], [], []
    covered = np.zeros(n, dtype=bool)
    for nd in sizes:
        idx = np.sort(perm[start:start + nd])
        start += nd
        q, _ = np.linalg.qr(rng.standard_normal((nd, nd)))
        blk = (q * np.logspace(0, -6, nd)) @ q.T
        blk = 0.5 * (blk + blk.T)
        r, c = np.meshgrid(idx, idx, indexing="ij")
        rows.append(r.ravel())
        cols.append(c.ravel())
        vals.append(blk.ravel())
        covered[idx] = True
        sets.append(idx)
    rest = np.nonzero(~covered)[0]
    rows.append(rest)
    cols.append(rest)
    vals.append(np.ones(len(rest)))
    a = sm.sparse.CsrMatrix.from_coo(n, n, np.concatenate(rows), np.concatenate(cols),
                                     np.concatenate(vals))
    lc = sm.smoothers.build_local_correction(a, sets)
    d = {"n": np.array(n)}
    for k, s in enumerate(sets):
        d[f"set{k}"] = s
    r = rng.standard_normal(n)
    d["r"] = r
    d["lc_apply"] = sm.smoothers.apply_local_correction(lc, r)
    for k, (idx, fac) in enumerate(lc.regions):
        c = fac.factor[0]
        d[f"ltri{k}"] = c[np.tril_indices(len(idx))]  # lower factor, row-major packed
    _versions(d)
    np.savez_compressed(fixtures.path("c5p"), **d)
    print("c5p", sizes)


def _coupling(a, regions):
    """1 if any two regions are coupled through A (A[B_d, B_d'] != 0)."""
    s = a.to_scipy()
    owner = -np.ones(a.nrows, dtype=np.int64)
    for k, (idx, _) in enumerate(regions):
        owner[idx] = k
    for k, (idx, _) in enumerate(regions):
        sub = s[idx]
        cols = sub.indices[sub.data != 0.0]
        o = owner[cols]
        if np.any((o >= 0) & (o != k)):
            return 1
    return 0


def multi_region(name, degree, centers, grids=(16, 8, 4), jacobi_theta=None, sweeps=2):
    """Several local-correction regions on the fine level, built entirely by
    the reference: structured grids (mesh.py:136), two or more flattened
    vertices by the reference's own cluster routine (experiments.py:175-263,
    one vertex per cluster, seeded), regions / dofs / factors / lambda by
    build_hierarchy (mg.py:72-124).  SURVEY.md A4: with the flattened vertices
    4 cells apart at n = 16 the two regions are disjoint but coupled through A
    (additive S_c must read the pre-correction u); far apart they are not."""
    sm = _ref()
    ex = sm.experiments
    meshes = []
    for lvl, n in enumerate(grids):
        m = sm.mesh.generate_simplex_grid(2, n)
        if lvl == 0:
            clusters = [ex.ClusterSpec(c, 1e-4, 1) for c in centers]
            m = ex._apply_clusters(m, clusters, np.random.default_rng([5, lvl]))
        meshes.append(m)
    zero = lambda x: 0.0
    problem = sm.fem.ProblemSpec("poisson", source=lambda x: 1.0,
                                 dirichlet=tuple((m, zero) for m in range(1, 5)))
    smoother = sm.smoothers.SmootherConfig("chebyshev", sweeps)
    h = sm.mg.build_hierarchy(meshes, problem, smoother, True, 0.1, degree)
    if jacobi_theta is not None:
        for lv in h.levels:
            lv.smoother = sm.smoothers.SmootherConfig("chebyshev", sweeps, lambda_max=jacobi_theta,
                                                      lambda_min_fraction=1.0)
    lv0 = h.levels[0]
    lc = lv0.local_correction
    n0 = lv0.a.nrows
    b = np.array(h.system.b)
    d = fixtures.hierarchy_arrays(h)
    _common_goldens(sm, h, b, np.zeros(n0), d)
    d["coupled"] = np.array(_coupling(lv0.a, lc.regions))
    d["lambda_max"] = np.array([lv.lambda_max for lv in h.levels])
    d["lambda_max_adjusted"] = np.array([lv.lambda_max_adjusted for lv in h.levels])
    d["meta/grids"] = np.array(grids)
    _versions(d)
    np.savez_compressed(fixtures.path(name), **d)
    print(name, [lv.a.nrows for lv in h.levels], "regions", lc.n_regions,
          [len(i) for i, _ in lc.regions], "coupled", int(d["coupled"]),
          "stat iters", int(d["g/stat_iters"]), "cg iters", int(d["g/cg_iters"]))


def main():
    t = time.time()
    which = set(sys.argv[1:])

    def want(name):
        return not which or name in which

    if want("crit7"):
        crit7()
    if want("c1s"):
        baseline_small("c1s", fixtures.workload("c1s"), jacobi_theta=1.5)
    if want("c2s"):
        baseline_small("c2s", fixtures.workload("c2s"), layers=2)
    if want("c3s"):
        baseline_small("c3s", fixtures.workload("c3s"), jacobi_theta=1.5)
    if want("c4s"):
        # BASELINE C4 construction (3D P2, jitter 0.15h, flattened tets,
        # Chebyshev degree 2) at grids 12/6/3/2 with two clusters: P2 patches
        # of ~200 dofs (SURVEY.md finding 6) on a 15,625-dof fine level
        baseline_small("c4s", fixtures.workload("c4s"))
    if want("c5p"):
        c5_patches()
    # multi-region local corrections (pkg/tests/test_smoothers.py:89-99)
    if want("cpl_p1"):
        multi_region("cpl_p1", 1, [(0.3125, 0.5), (0.5625, 0.5)], jacobi_theta=1.5)
    if want("cpl_p2"):
        multi_region("cpl_p2", 2, [(0.3125, 0.5), (0.5625, 0.5)])
    if want("unc_p2"):
        multi_region("unc_p2", 2, [(0.25, 0.25), (0.75, 0.75), (0.25, 0.75)])
    print(f"done in {time.time() - t:.1f}s")


if __name__ == "__main__":
    main()
