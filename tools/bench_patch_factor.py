"""Time the batched device Cholesky of local-correction blocks (smg_patch_factor)
against the reference's per-block scipy cho_factor (smoothers.py:176-200), on
BASELINE C5's patch population: 1000 SPD blocks of 64-512 DOFs, cond 1e6
(SURVEY.md 8(d)), embedded block-diagonally in a sparse operator.

    python tools/bench_patch_factor.py [--patches 1000] [--out FILE]
"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    npatch = int(sys.argv[sys.argv.index("--patches") + 1]) if "--patches" in sys.argv else 1000
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    import scipy.sparse as sp
    import torch
    from paper_2402_12947_b200.smoothers import build_local_correction
    from paper_2402_12947_b200.sparse import CsrMatrix
    rng = np.random.default_rng(2024)
    sizes = rng.integers(64, 513, size=npatch)
    n = int(sizes.sum())
    offs = np.concatenate([[0], np.cumsum(sizes)])
    rows, cols, vals = [], [], []
    sets = []
    for k, nd in enumerate(sizes):
        q, _ = np.linalg.qr(rng.standard_normal((nd, nd)))
        b = (q * np.logspace(0, -6, nd)) @ q.T
        b = 0.5 * (b + b.T)
        idx = np.arange(offs[k], offs[k + 1])
        ii, jj = np.meshgrid(idx, idx, indexing="ij")
        rows.append(ii.ravel()); cols.append(jj.ravel()); vals.append(b.ravel())
        sets.append(idx)
    a = CsrMatrix.from_scipy(sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows),
                                            np.concatenate(cols))), shape=(n, n)).tocsr())
    build_local_correction(a, sets[:4], device=True)  # upload + warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev = build_local_correction(a, sets, device=True)
    gpu_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    host = build_local_correction(a, sets, device=False)
    cpu_s = time.perf_counter() - t0
    worst = 0.0
    for (_, fd), (_, fh) in zip(dev.regions, host.regions):
        ld, lh = np.tril(fd.factor[0]), np.tril(fh.factor[0])
        worst = max(worst, float(np.max(np.abs(ld - lh)) / np.max(np.abs(lh))))
    flops = float(np.sum(sizes.astype(np.float64) ** 3) / 3.0)
    rec = {"patches": npatch, "dofs": n, "factor_doubles": int(np.sum(sizes ** 2)),
           "gpu_ms": gpu_s * 1e3, "cpu_ms": cpu_s * 1e3, "speedup": cpu_s / gpu_s,
           "gpu_gflops_incl_copies": flops / gpu_s / 1e9, "max_rel_L_diff_vs_lapack": worst,
           "cpu_threads": os.cpu_count()}
    print(json.dumps(rec), flush=True)
    if out:
        with open(out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
