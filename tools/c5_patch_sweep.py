"""Batched patch solve (smg_apply_local_correction) timing vs patch-size mix.

    python tools/c5_patch_sweep.py            # on the GPU box

Cases: BASELINE C5's 1000 patches of U[64, 512] dofs (cond 1e6), then
uniform sizes (64 .. 512) with 1 patch (the single-patch latency = the
critical path of the largest region) and 1000 patches (throughput).  Prints
one JSON line per case: us per application, factor bytes, GB/s."""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def make(sizes, n_rows, seed=7):
    import torch
    from paper_2402_12947_b200.smoothers import LocalCorrection
    from paper_2402_12947_b200.sparse import DenseFactor
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n_rows)
    g = torch.Generator(device="cuda").manual_seed(seed)
    cache = {}
    regions, start = [], 0
    for nd in sizes:
        nd = int(nd)
        idx = np.sort(perm[start:start + nd])
        start += nd
        if nd not in cache:
            q, _ = torch.linalg.qr(torch.randn(nd, nd, dtype=torch.float64, device="cuda",
                                               generator=g))
            lam = torch.logspace(0, -6, nd, dtype=torch.float64, device="cuda")
            blk = (q * lam) @ q.T
            blk = 0.5 * (blk + blk.T)
            cache[nd] = torch.linalg.cholesky(blk).cpu().numpy()
        regions.append((idx.astype(np.int64), DenseFactor("cholesky", (cache[nd], True), nd)))
    return LocalCorrection(tuple(regions), n_rows)


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default=None, help="run only this case (e.g. '512 x1', 'C5')")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_2402_12947_b200 import _lib, device as D
    from paper_2402_12947_b200.sparse import CsrMatrix
    torch.cuda.set_device(0)
    lib = _lib.load()
    n = 600_000
    op = D.DeviceOperator(CsrMatrix.identity(n))
    r = torch.randn(n, dtype=torch.float64, device="cuda")
    o = torch.empty_like(r)
    sh = D.stream_handle()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cases = [("C5 U[64,512] x1000", np.random.default_rng(2402).integers(64, 513, size=1000))]
    for nd in (64, 128, 192, 256, 384, 512):
        cases.append((f"{nd} x1", np.array([nd])))
        cases.append((f"{nd} x1000", np.full(1000, nd)))
    if args.case:
        cases = [(nm, sz) for nm, sz in cases if nm.startswith(args.case)]
    for name, sizes in cases:
        lc = make(sizes, n)
        dc = D.DeviceCorrection(op, lc)
        for _ in range(3):
            _lib.check(lib.smg_apply_local_correction(dc.handle, D.ptr(r), D.ptr(o), sh))
        torch.cuda.synchronize()
        reps = args.reps
        e0.record()
        for _ in range(reps):
            _lib.check(lib.smg_apply_local_correction(dc.handle, D.ptr(r), D.ptr(o), sh))
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        fb = float(np.sum(8.0 * sizes * (sizes + 1) / 2))
        print(json.dumps({"case": name, "us": round(us, 2), "factor_MB": round(fb / 1e6, 2),
                          "single_pass_GBs": round(fb / us / 1e3, 1),
                          "env": {k: v for k, v in os.environ.items() if k.startswith("SMG_")}}),
              flush=True)
        del dc


if __name__ == "__main__":
    main()
