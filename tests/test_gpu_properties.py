"""Property tests of the GPU path, restating the reference suite's dense
checks (pkg/tests/test_smoothers.py, test_mg.py) at small sizes.

All operators are materialised by applying the GPU smoother / V-cycle to
unit vectors through the C-ABI, then compared with closed forms:
  * Chebyshev error propagation = T_k(Z)/T_k(sigma) (test_smoothers.py:175-201), 1e-10;
  * sandwich operator = 2S_c - S_c A S_c + (I - S_c A) S_g (I - A S_c)
    (test_smoothers.py:295-305), 1e-11, and symmetric (:307-318);
  * V-cycle: zero is a fixed point, identical meshes are exact in one cycle,
    the preconditioner is symmetric (test_mg.py:105-130, :194-208), and CG
    with it decreases the energy error monotonically (:216-240).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def random_spd(n, seed):
    rng = np.random.default_rng(seed)
    m = rng.standard_normal((n, n))
    return m @ m.T + n * np.eye(n)


def sparse_spd(n, seed, band=3):
    """Banded SPD matrix (diagonally dominant) as a CsrMatrix."""
    from paper_2402_12947_b200.sparse import CsrMatrix
    rng = np.random.default_rng(seed)
    a = np.zeros((n, n))
    for k in range(1, band + 1):
        v = rng.uniform(-1, 1, n - k)
        a += np.diag(v, k) + np.diag(v, -k)
    a += np.diag(2.0 * band + rng.uniform(1, 2, n))
    return CsrMatrix.from_dense(a), a


def smoother_matrix(apply, n):
    """Columns: apply(e_j) for the linear map e -> apply(e)."""
    return np.column_stack([apply(np.eye(n)[:, j]) for j in range(n)])


def test_chebyshev_error_propagation_is_the_minimax_polynomial():
    import paper_2402_12947_b200 as P
    from numpy.polynomial import chebyshev as C
    n, k = 30, 3
    a_csr, a = sparse_spd(n, 1)
    d = np.diag(a)
    dinv_half = 1.0 / np.sqrt(d)
    s = dinv_half[:, None] * a * dinv_half[None, :]
    lam_max = float(np.linalg.eigvalsh(s).max())
    cfg = P.SmootherConfig("chebyshev", k, lambda_max=lam_max, lambda_min_fraction=0.1)

    def err(e0):  # b = 0: the iterate is the error
        u = e0.copy()
        P.chebyshev_smooth(a_csr, np.zeros(n), u, k, cfg)
        return u

    m = smoother_matrix(err, n)
    lam_min = 0.1 * lam_max
    theta, delta = 0.5 * (lam_max + lam_min), 0.5 * (lam_max - lam_min)
    w, v = np.linalg.eigh(s)
    coef = np.zeros(k + 1)
    coef[k] = 1.0
    p = C.chebval((theta - w) / delta, coef) / C.chebval(theta / delta, coef)
    expected = dinv_half[:, None] * (v * p) @ v.T / dinv_half[None, :]
    np.testing.assert_allclose(m, expected, atol=1e-10 * np.abs(expected).max())


def _region_setup(n, seed):
    import paper_2402_12947_b200 as P
    a_csr, a = sparse_spd(n, seed)
    rng = np.random.default_rng(seed + 1)
    perm = rng.permutation(n)
    sets = [np.sort(perm[:6]), np.sort(perm[10:17])]
    lc = P.build_local_correction(a_csr, sets)
    sc = np.zeros((n, n))
    for idx in sets:
        sc[np.ix_(idx, idx)] = np.linalg.inv(a[np.ix_(idx, idx)])
    return a_csr, a, lc, sc


def test_sandwich_operator_matches_dense_formula_and_is_symmetric():
    import paper_2402_12947_b200 as P
    n = 32
    a_csr, a, lc, sc = _region_setup(n, 3)
    d = np.diag(a)
    lam = float(np.linalg.eigvalsh(a / np.sqrt(np.outer(d, d))).max())
    cfg = P.SmootherConfig("chebyshev", 3, lambda_max=lam)

    def comb(r):  # b = r, u = 0: the combined smoother as a map r -> u
        u = np.zeros(n)
        P.combined_smooth(a_csr, r, u, lc, cfg)
        return u

    def glob(r):
        u = np.zeros(n)
        P.chebyshev_smooth(a_csr, r, u, 3, cfg)
        return u

    s_gc = smoother_matrix(comb, n)
    s_g = smoother_matrix(glob, n)
    eye = np.eye(n)
    expected = 2 * sc - sc @ a @ sc + (eye - sc @ a) @ s_g @ (eye - a @ sc)
    np.testing.assert_allclose(s_gc, expected, atol=1e-11 * np.abs(expected).max())
    assert np.abs(s_gc - s_gc.T).max() <= 1e-11 * np.abs(s_gc).max()


def _two_level_identity(a_csr, a, smoother):
    """A hierarchy whose coarse level is the fine one (P = I): exact in one cycle."""
    import paper_2402_12947_b200 as P
    from paper_2402_12947_b200.mg import Hierarchy, Level, Prolongation
    from paper_2402_12947_b200.sparse import CsrMatrix
    n = a.shape[0]
    eye = CsrMatrix.identity(n)
    levels = [Level(0, None, None, a_csr, Prolongation(eye, 0, 1), smoother, None, None),
              Level(1, None, None, a_csr, None, smoother, None, None)]
    return Hierarchy(levels, P.dense_factor(a))


def test_vcycle_fixed_points_and_identical_meshes_exact():
    import paper_2402_12947_b200 as P
    n = 40
    a_csr, a = sparse_spd(n, 5)
    cfg = P.SmootherConfig("chebyshev", 2, lambda_max=2.0)
    h = _two_level_identity(a_csr, a, cfg)
    u = np.zeros(n)
    P.vcycle(h, np.zeros(n), u)
    assert np.all(u == 0.0)
    b = np.random.default_rng(0).standard_normal(n)
    u = np.zeros(n)
    P.vcycle(h, b, u)
    np.testing.assert_allclose(a @ u, b, rtol=0, atol=1e-10 * np.abs(b).max())


def test_preconditioner_symmetric_and_cg_energy_monotone():
    import paper_2402_12947_b200 as P
    from tests.golden import fixtures
    z, h = fixtures.load("c1s")
    a = h.levels[0].a.to_dense()
    n = a.shape[0]
    pre = P.as_preconditioner(h)
    rng = np.random.default_rng(3)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    bx, by = pre(x), pre(y)
    assert abs(x @ by - y @ bx) <= 1e-10 * max(abs(x @ by), 1.0)
    # CG energy error decreases monotonically (test_mg.py:216-240)
    b = z["g/b"]
    xs = np.linalg.solve(a, b)
    errs = []
    for it in range(1, 7):
        xk, _ = P.cg(h.levels[0].a, b, precond=pre, rtol=0.0, maxit=it)
        e = xk - xs
        errs.append(float(e @ a @ e))
    assert all(e2 <= e1 * (1 + 1e-12) for e1, e2 in zip(errs, errs[1:]))
