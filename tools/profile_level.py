"""Back-to-back smoother steps on one level of a workload, for a WARM ncu
capture (--cache-control none; the operator stays L2-resident between the
launches, as it does inside a V-cycle for the small levels).

    ncu --cache-control none --clock-control none --set full -k regex:csr_tile_kernel \
        --launch-skip 4 --launch-count 1 python tools/profile_level.py --level 2
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--level", type=int, default=2)
    ap.add_argument("--reps", type=int, default=6)
    args = ap.parse_args()
    import torch
    from paper_2402_12947_b200 import _lib, configs, device as D
    h, _, _ = configs.build(configs.WORKLOADS[args.workload])
    lv = h.levels[args.level]
    op = D.device_operator(lv.a)
    lib = _lib.load()
    n = op.nrows
    xa = torch.randn(n, dtype=torch.float64, device="cuda")
    xb = torch.empty_like(xa)
    d = torch.zeros_like(xa)
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    lam = float(lv.smoother.chebyshev_parameters()[0]) if hasattr(lv.smoother, "chebyshev_parameters") \
        else float(lv.smoother.lambda_max)
    for _ in range(args.reps):
        _lib.check(lib.smg_smoother_step(op.handle, D.ptr(b), D.ptr(xa), D.ptr(xb), D.ptr(d), 2,
                                         0.55 * lam, 0.3, 0.7, D.stream_handle()))
        xa, xb = xb, xa
    torch.cuda.synchronize()
    print("ok", n, op.nnz)


if __name__ == "__main__":
    main()
