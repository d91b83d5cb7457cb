"""CPU study behind the symmetric-inverse patch path: how far x = A^-1 r and
x = L^-T (L^-1 r) are from the reference's cho_solve, and all three from a
refined solution, on every local-correction region of the golden fixtures and
on the cond-1e6 C5 blocks.  numpy/scipy only (run here, no GPU).

    python profiles/r02/sym/accuracy_study.py > profiles/r02/sym/accuracy_study.txt
"""
import os
import sys

import numpy as np
import scipy.linalg as sl
import scipy.sparse as sp

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", ".."))
from tests.golden import fixtures  # noqa: E402


def study(name, blk, c, r):
    nd = len(r)
    L = np.tril(c)
    x = sl.cho_solve((c, True), r)
    Li = sl.solve_triangular(L, np.eye(nd), lower=True)
    x_linv = Li.T @ (Li @ r)
    x_ainv = (Li.T @ Li) @ r
    xr = x.astype(np.longdouble)
    for _ in range(3):
        res = r.astype(np.longdouble) - blk.astype(np.longdouble) @ xr
        xr = xr + sl.cho_solve((c, True), res.astype(np.float64))
    f = lambda v: float(np.linalg.norm(v - x) / np.linalg.norm(x))      # noqa: E731
    g = lambda v: float(np.linalg.norm(v - xr) / np.linalg.norm(xr))    # noqa: E731
    print(f"{name} n={nd} cond={np.linalg.cond(blk):.2e} | vs cho_solve: Linv {f(x_linv):.1e} "
          f"Ainv {f(x_ainv):.1e} | vs refined: cho_solve {g(x):.1e} Linv {g(x_linv):.1e} "
          f"Ainv {g(x_ainv):.1e}")


def main():
    rng = np.random.default_rng(0)
    for name in ["c1s", "c2s", "c3s", "c4s", "cpl_p1", "cpl_p2", "unc_p2", "crit7_adj"]:
        z, h = fixtures.load(name)
        for l, lv in enumerate(h.levels):
            lc = lv.local_correction
            if lc is None:
                continue
            a = lv.a
            m = sp.csr_matrix((a.values, a.col_indices, a.row_offsets), shape=(a.nrows, a.ncols))
            for k, (idx, fac) in enumerate(lc.regions):
                c, _ = fac.factor
                u = rng.standard_normal(a.nrows)
                b = rng.standard_normal(a.nrows)
                r = (b - m @ u)[idx]
                study(f"{name} L{l} R{k}", m[idx][:, idx].toarray(), c, r)
    rng = np.random.default_rng(2402)
    for nd in [64, 200, 512]:
        q, _ = np.linalg.qr(rng.standard_normal((nd, nd)))
        blk = (q * np.logspace(0, -6, nd)) @ q.T
        blk = 0.5 * (blk + blk.T)
        c = sl.cho_factor(blk, lower=True)[0]
        study(f"C5-style cond-1e6 block", blk, c, rng.standard_normal(nd))


if __name__ == "__main__":
    main()
