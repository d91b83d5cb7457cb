"""Golden-fixture (de)serialisation: hierarchies and reference outputs as .npz.

A fixture stores a multigrid hierarchy exactly as the reference built it
(CSR arrays of every A_l and P_l, region dof sets with their Cholesky factors
``c`` from scipy cho_factor, smoother parameters, the coarse factor) plus the
reference's outputs on seeded inputs.  Loading rebuilds
``paper_2402_12947_b200`` host objects, which the GPU path and the oracle
both accept.
"""

from __future__ import annotations

import os
from typing import Dict

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def path(name: str) -> str:
    return os.path.join(HERE, name + ".npz")


def _put_csr(d: Dict, key: str, m) -> None:
    d[key + "/shape"] = np.array([m.nrows, m.ncols], dtype=np.int64)
    d[key + "/ptr"] = np.asarray(m.row_offsets, dtype=np.int64)
    d[key + "/col"] = np.asarray(m.col_indices, dtype=np.int64)
    d[key + "/val"] = np.asarray(m.values, dtype=np.float64)


def _get_csr(z, key: str):
    from paper_2402_12947_b200.sparse import CsrMatrix
    nr, nc = (int(v) for v in z[key + "/shape"])
    return CsrMatrix(nr, nc, z[key + "/ptr"], z[key + "/col"], z[key + "/val"])


def hierarchy_arrays(h, prefix: str = "h") -> Dict[str, np.ndarray]:
    """Serialise a reference (or product) Hierarchy."""
    d = {}
    nl = len(h.levels)
    d[prefix + "/n_levels"] = np.array(nl)
    for l, lv in enumerate(h.levels):
        p = f"{prefix}/L{l}"
        _put_csr(d, p + "/a", lv.a)
        if lv.prolongation is not None:
            _put_csr(d, p + "/p", lv.prolongation.matrix)
        cfg = lv.smoother
        d[p + "/cfg"] = np.array([cfg.sweeps, cfg.lambda_max if cfg.lambda_max is not None else -1.0,
                                  cfg.lambda_min_fraction], dtype=np.float64)
        d[p + "/kind"] = np.array(cfg.kind)
        lc = lv.local_correction
        nreg = 0 if lc is None else len(lc.regions)
        d[p + "/n_regions"] = np.array(nreg)
        for k in range(nreg):
            idx, fac = lc.regions[k]
            c, lower = fac.factor
            assert lower
            d[p + f"/R{k}/idx"] = np.asarray(idx, dtype=np.int64)
            d[p + f"/R{k}/c"] = np.asarray(c, dtype=np.float64)
    c, lower = h.coarse_factor.factor
    assert lower and h.coarse_factor.kind == "cholesky"
    d[prefix + "/coarse_c"] = np.asarray(c, dtype=np.float64)
    return d


def load_hierarchy(z, prefix: str = "h"):
    """Rebuild product host objects from a fixture."""
    from paper_2402_12947_b200.mg import Hierarchy, Level, Prolongation
    from paper_2402_12947_b200.smoothers import LocalCorrection, SmootherConfig
    from paper_2402_12947_b200.sparse import DenseFactor
    nl = int(z[prefix + "/n_levels"])
    levels = []
    for l in range(nl):
        p = f"{prefix}/L{l}"
        a = _get_csr(z, p + "/a")
        prol = Prolongation(_get_csr(z, p + "/p"), l, l + 1) if (p + "/p/shape") in z else None
        sweeps, lam, frac = z[p + "/cfg"]
        kind = str(z[p + "/kind"])
        cfg = SmootherConfig(kind, int(sweeps), None if lam < 0 else float(lam), float(frac))
        nreg = int(z[p + "/n_regions"])
        lc = None
        if nreg:
            regs = []
            for k in range(nreg):
                idx = z[p + f"/R{k}/idx"]
                c = z[p + f"/R{k}/c"]
                regs.append((idx, DenseFactor("cholesky", (c, True), len(idx))))
            lc = LocalCorrection(tuple(regs), a.nrows)
        levels.append(Level(l, None, None, a, prol, cfg, None, lc))
    c = z[prefix + "/coarse_c"]
    return Hierarchy(levels, DenseFactor("cholesky", (c, True), c.shape[0]))


def load(name: str):
    """Open a fixture: returns (npz mapping, hierarchy or None)."""
    z = dict(np.load(path(name), allow_pickle=False))
    h = load_hierarchy(z) if "h/n_levels" in z else None
    return z, h


#: every fixture that stores a whole reference-built hierarchy and its outputs
HIERARCHY_FIXTURES = ["crit7_adj", "crit7_ref", "c1s", "c2s", "c3s", "c4s",
                      "cpl_p1", "cpl_p2", "unc_p2"]
#: fixtures whose fine level holds several local-correction regions, and
#: whether those regions are coupled through A
MULTI_REGION_FIXTURES = {"cpl_p1": True, "cpl_p2": True, "unc_p2": False}


def workload(name: str):
    """The paper_2402_12947_b200.configs construction a baseline fixture was
    generated from (tests/golden/make_golden.py ``baseline_small``)."""
    from dataclasses import replace
    from paper_2402_12947_b200 import configs
    return {
        "c1s": configs.C1.scaled(4),
        "c2s": configs.C2.scaled(8),
        "c3s": configs.C3.scaled(4),
        "c4s": replace(configs.C4, name="C4-3d-p2-cheb2/s", grids=(12, 6, 3, 2), n_clusters=2),
    }[name]
