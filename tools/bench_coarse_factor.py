"""Time the coarse factor + inverse on the device (smg_dense_cholesky +
smg_cholesky_inverse: the hand-written blocked dpotrf / dtrtri / dlauum of
csrc/coarse_factor.cu) against scipy cho_factor + LAPACK dpotri on
the host, for a dense SPD matrix of the coarsest-level size of a workload
(C4: n_L = 15,625; the reference's mg.py:123 plus this package's A_L^-1).

    python tools/bench_coarse_factor.py [n] [--out FILE]
"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    args = [a for a in args if a != out]
    n = int(args[0]) if args else 15625
    import scipy.linalg
    import torch
    from paper_2402_12947_b200.mg import coarse_inverse
    from paper_2402_12947_b200.sparse import dense_factor
    rng = np.random.default_rng(0)
    g = rng.standard_normal((n, n)) / np.sqrt(n)
    a = g @ g.T + np.eye(n)
    dense_factor(a[:64, :64].copy(), device=True)  # warm-up (context, kernel attributes)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = dense_factor(a, device=True)
    t1 = time.perf_counter()
    inv_d = coarse_inverse(f, device=True)
    t2 = time.perf_counter()
    c = scipy.linalg.cho_factor(a, lower=True, check_finite=False)
    t3 = time.perf_counter()
    inv_h = coarse_inverse(c, device=False) if False else None
    lo = np.asfortranarray(np.tril(c[0]))
    inv_lapack, _ = scipy.linalg.lapack.dpotri(lo, lower=1)
    t4 = time.perf_counter()
    inv_lapack = np.tril(inv_lapack) + np.tril(inv_lapack, -1).T
    inv_rel = float(np.max(np.abs(inv_d - inv_lapack)) / np.max(np.abs(inv_lapack)))
    rel = float(np.max(np.abs(np.tril(f.factor[0]) - np.tril(c[0]))) / np.max(np.abs(np.tril(c[0]))))
    rec = {"n": n, "gpu_factor_ms": (t1 - t0) * 1e3, "gpu_inverse_ms": (t2 - t1) * 1e3,
           "cpu_factor_ms": (t3 - t2) * 1e3, "cpu_inverse_ms": (t4 - t3) * 1e3,
           "max_rel_L_diff": rel, "max_rel_inverse_diff": inv_rel,
           "gpu_includes": "H2D + hand-written kernels + D2H of n^2 doubles",
           "cpu_threads": os.cpu_count()}
    print(json.dumps(rec), flush=True)
    if out:
        with open(out, "w") as fo:
            json.dump(rec, fo, indent=1)


if __name__ == "__main__":
    main()
