"""GPU Galerkin coarse operators (smg_galerkin / smg_matmul) against the
reference's own coarse operators and the oracle.

Reference: sparse.py:147-154 triple_product (``ps.T @ (a @ ps)``), reached from
transfer.py:153-155 coarsen_system in mg.py:100 (setup).
Bar: BITWISE -- identical row offsets, column indices and values (the device
sums every entry in scipy csr_matmat's order and drops exact zeros as it does).
"""

import numpy as np
import pytest

from tests.golden import fixtures

from tests.test_oracle_golden import random_int_csr

pytestmark = pytest.mark.gpu

NAMES = fixtures.HIERARCHY_FIXTURES


def same(m, ptr, col, val) -> bool:
    return (np.array_equal(m.row_offsets, ptr) and np.array_equal(m.col_indices, col)
            and np.array_equal(m.values, val))


@pytest.mark.parametrize("name", NAMES)
def test_galerkin_bitwise_vs_reference(name):
    from paper_2402_12947_b200.sparse import triple_product
    from tests.golden import fixtures
    z, h = fixtures.load(name)
    for l in range(len(h.levels) - 1):
        lv = h.levels[l]
        c = triple_product(lv.prolongation.matrix, lv.a)
        ref = h.levels[l + 1].a
        assert same(c, ref.row_offsets, ref.col_indices, ref.values), f"{name} level {l + 1}"


def test_matmul_vs_oracle_cancellations_empty_rows():
    from oracle import oracle as O
    from paper_2402_12947_b200.sparse import matmul
    rng = np.random.default_rng(11)
    for (n, k, m, d) in [(40, 30, 50, 0.2), (7, 300, 9, 0.5), (200, 150, 120, 0.05),
                         (1, 1, 1, 1.0)]:
        x = random_int_csr(rng, n, k, d, empty_rows=(0,) if n > 1 else ())
        y = random_int_csr(rng, k, m, d)
        c = matmul(x, y)
        assert same(c, *O.spgemm(x, y))
        assert np.all(c.values != 0.0)
    xf = random_int_csr(rng, 300, 400, 0.05, values=tuple(rng.standard_normal(32)))
    yf = random_int_csr(rng, 400, 350, 0.05, values=tuple(rng.standard_normal(32)))
    assert same(matmul(xf, yf), *O.spgemm(xf, yf))


def test_matmul_long_rows_take_the_cta_paths():
    """Rows with > 512 unique columns (CTA numeric path) and > 1024 (CTA
    recount after the warp table overflows), mixed with short rows."""
    from oracle import oracle as O
    from paper_2402_12947_b200.sparse import CsrMatrix, matmul
    rng = np.random.default_rng(3)
    ncols = 5000
    y = random_int_csr(rng, 400, ncols, 0.004, values=tuple(rng.standard_normal(8)))
    dense_rows = {3: 30, 10: 200, 17: 400}      # X row -> entries (many Y rows each)
    rows, cols = [], []
    for r in range(24):
        k = dense_rows.get(r, 2)
        cs = np.sort(rng.choice(400, size=k, replace=False))
        rows += [r] * k
        cols += list(cs)
    x = CsrMatrix.from_coo(24, 400, np.array(rows), np.array(cols), rng.standard_normal(len(rows)))
    c = matmul(x, y)
    lens = np.diff(c.row_offsets)
    assert lens[17] > 1024 and lens[10] > 1024 and 512 < lens[3] <= 1024
    assert same(c, *O.spgemm(x, y))


def test_empty_and_zero_products():
    from paper_2402_12947_b200.sparse import CsrMatrix, matmul
    e = CsrMatrix(5, 4, np.zeros(6, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros(0))
    y = CsrMatrix.from_dense(np.ones((4, 3)))
    c = matmul(e, y)
    assert c.shape == (5, 3) and c.nnz == 0 and np.array_equal(c.row_offsets, np.zeros(6))
    # every product cancels: explicit zero sums are dropped (csr_matmat)
    x = CsrMatrix.from_dense(np.array([[1.0, -1.0]]))
    y = CsrMatrix.from_dense(np.array([[2.0, 3.0], [2.0, 3.0]]))
    c = matmul(x, y)
    assert c.nnz == 0 and np.array_equal(c.row_offsets, [0, 0])


def test_galerkin_errors():
    from paper_2402_12947_b200.sparse import CsrMatrix, matmul, triple_product
    a = CsrMatrix.from_dense(np.eye(4))
    p = CsrMatrix.from_dense(np.ones((3, 2)))
    with pytest.raises(ValueError, match="dimension mismatch"):
        triple_product(p, a)
    with pytest.raises(ValueError, match="dimension mismatch"):
        matmul(a, p)


@pytest.mark.slow
def test_galerkin_full_size_c2_bitwise():
    """Full BASELINE C2 hierarchy (1.05M fine DOFs, 5 levels): every device
    Galerkin operator equals the reference's scipy product bit for bit."""
    from paper_2402_12947_b200 import configs
    from paper_2402_12947_b200.sparse import host_triple_product, triple_product
    h = configs.build(configs.C2)[0]
    for l in range(len(h.levels) - 1):
        lv = h.levels[l]
        ref = host_triple_product(lv.prolongation.matrix, lv.a)
        c = triple_product(lv.prolongation.matrix, lv.a)
        assert same(c, ref.row_offsets, ref.col_indices, ref.values), f"level {l + 1}"
