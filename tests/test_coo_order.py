"""scipy's COO -> CSR duplicate order, as the device reproduces it (CPU test).

fem.py:339-345 assembles with coo_matrix(...).tocsr(); scipy buckets the
entries by row in input order and, unless every row is already sorted, runs
libstdc++'s std::sort on each row's (column, value) pairs comparing columns
only, then adds runs of equal columns in the resulting order.
smg_assemble_elements (paper_2402_12947_b200/csrc/coo_kernels.cu) restates
that sort for one thread per row.  This test builds the same __host__
__device__ code for the host (tests/native/coo_sort_host.cu, nvcc) and checks
it against libstdc++'s own std::sort and against scipy itself, including
McIlroy's antiqsort adversary (quicksort depth limit -> heapsort fallback).
The device pipeline as a whole is checked against scipy in
tests/test_gpu_setup.py::test_scipy_order_duplicate_sums.
"""

import ctypes
import os
import shutil
import subprocess

import numpy as np
import pytest
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    if not (os.path.exists(NVCC) or shutil.which("nvcc")):
        pytest.skip("nvcc not available")
    out = str(tmp_path_factory.mktemp("coo") / "libcoo_sort_host.so")
    src = os.path.join(HERE, "native", "coo_sort_host.cu")
    subprocess.run([NVCC, "-std=c++17", "-O2", "-Xcompiler", "-fPIC,-ffp-contract=off",
                    "-shared", "-o", out, src], check=True, capture_output=True)
    lb = ctypes.CDLL(out)
    i32p, f64p = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double)
    for name in ("emulated_row_sort", "libstdcxx_row_sort"):
        getattr(lb, name).argtypes = [ctypes.c_int64, i32p, f64p]
    lb.antiqsort_input.argtypes = [ctypes.c_int64, i32p]
    return lb


def _sorted(fn, cols, vals):
    c = np.ascontiguousarray(cols, dtype=np.int32).copy()
    v = np.ascontiguousarray(vals, dtype=np.float64).copy()
    fn(len(c), c.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
       v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return c, v


def _runs(c, v):
    oc, ov = [], []
    j = 0
    while j < len(c):
        cc, x = c[j], v[j]
        j += 1
        while j < len(c) and c[j] == cc:
            x += v[j]
            j += 1
        oc.append(cc)
        ov.append(x)
    return np.array(oc, dtype=np.int64), np.array(ov)


def test_matches_scipy_on_random_rows(lib):
    g = np.random.default_rng(3)
    for t in range(1500):
        m = int(g.integers(1, 500))
        nc = int(g.integers(1, 60))
        cols = g.integers(0, nc, size=m)
        if t % 5 == 0:
            cols = np.sort(cols)[::-1].copy()
        vals = g.standard_normal(m) * 10.0 ** g.integers(-8, 8, size=m)
        # a second, unsorted row makes scipy sort every row
        a = sp.coo_matrix((np.r_[vals, [1.0, 1.0]], (np.r_[np.zeros(m, int), [1, 1]],
                                                     np.r_[cols, [1, 0]])), shape=(2, 64)).tocsr()
        a.sum_duplicates()
        c, v = _runs(*_sorted(lib.emulated_row_sort, cols, vals))
        assert np.array_equal(a.indices[:a.indptr[1]], c), t
        assert np.array_equal(a.data[:a.indptr[1]], v), t


@pytest.mark.parametrize("n", [17, 64, 200, 1000, 5000])
def test_matches_libstdcxx_on_antiqsort_and_duplicates(lib, n):
    """Identical permutations (columns and the values riding along) to the
    real std::sort on an adversarial input -- this one exhausts the 2 log2 n
    partition budget, so the heapsort fallback runs -- and on heavy-duplicate
    inputs."""
    keys = np.zeros(n, dtype=np.int32)
    lib.antiqsort_input(n, keys.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    vals = np.arange(n, dtype=np.float64)     # tags: any permutation difference shows
    for cols in (keys, keys % 7, np.zeros(n, dtype=np.int32), (keys * 31) % 13):
        c1, v1 = _sorted(lib.emulated_row_sort, cols, vals)
        c2, v2 = _sorted(lib.libstdcxx_row_sort, cols, vals)
        assert np.array_equal(c1, c2) and np.array_equal(v1, v2)
