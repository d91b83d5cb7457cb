"""Full-size parity record: GPU path vs the CPU oracle on one BASELINE workload.

    python tools/parity_fullsize.py --workload C4 > profiles/r01/parity_C4.json

Builds the workload's hierarchy (seeded), then on identical inputs compares:
  * every fine-level smoother sweep (bitwise), restriction / prolongation
    (bitwise) on every level;
  * one V-cycle from a random iterate (relative l2 difference);
  * stationary solve to 1e-10 (iteration counts and histories).
Prints one JSON object.  Test infrastructure (imports oracle/).
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--max-cycles", type=int, default=60)
    args = ap.parse_args()
    import torch
    import paper_2402_12947_b200 as P
    from paper_2402_12947_b200 import _lib, configs, device as D
    from oracle import oracle as O
    O.set_threads(len(os.sched_getaffinity(0)))
    t0 = time.perf_counter()
    h, b, u0 = configs.build(configs.WORKLOADS[args.workload])
    out = {"workload": args.workload, "setup_s": time.perf_counter() - t0,
           "levels_dofs": [lv.a.nrows for lv in h.levels]}
    lv = h.levels[0]
    ur = np.random.default_rng(5).standard_normal(lv.a.nrows)
    sweeps = []
    for k in range(1, lv.smoother.sweeps + 1):
        u = ur.copy()
        P.chebyshev_smooth(lv.a, b, u, k, lv.smoother)
        cfg = type(lv.smoother)(lv.smoother.kind, k, lv.smoother.lambda_max,
                                lv.smoother.lambda_min_fraction, omega=lv.smoother.omega)
        sweeps.append(bool(np.array_equal(u, O.global_smooth(lv.a, b, ur.copy(), cfg))))
    out["fine_sweeps_bitwise"] = sweeps
    lib = _lib.load()
    # every non-coarse level: one smoother call of the level's degree and the
    # residual, bitwise, with the layout the level's sweeps run on
    levels = []
    for l, lvl in enumerate(h.levels[:-1]):
        n = lvl.a.nrows
        ul = np.random.default_rng(200 + l).standard_normal(n)
        bl = np.random.default_rng(300 + l).standard_normal(n)
        ug = ul.copy()
        P.chebyshev_smooth(lvl.a, bl, ug, lvl.smoother.sweeps, lvl.smoother)
        ok_s = bool(np.array_equal(ug, O.global_smooth(lvl.a, bl, ul.copy(), lvl.smoother)))
        op = D.device_operator(lvl.a)
        bt, ut = torch.from_numpy(bl).cuda(), torch.from_numpy(ul).cuda()
        rt = torch.empty_like(bt)
        _lib.check(lib.smg_residual(op.handle, D.ptr(bt), D.ptr(ut), D.ptr(rt), D.stream_handle()))
        ok_r = bool(np.array_equal(rt.cpu().numpy(), bl - O.spmv(lvl.a, ul)))
        import ctypes
        lay, unr = ctypes.c_int(), ctypes.c_int()
        _lib.check(lib.smg_operator_layout(op.handle, ctypes.byref(lay), ctypes.byref(unr)))
        levels.append({"level": l, "rows": n, "nnz": lvl.a.nnz,
                       "layout": ["tiles", "tiles-fixed", "sell", "sell4", "sell-d16"][lay.value], "unroll": unr.value,
                       "smooth_bitwise": ok_s, "residual_bitwise": ok_r})
    out["levels"] = levels
    transfers = []
    for l, lvl in enumerate(h.levels[:-1]):
        pm = lvl.prolongation.matrix
        op = D.device_operator(pm, with_transpose=True)
        r = np.random.default_rng(l).standard_normal(pm.nrows)
        uc = np.random.default_rng(100 + l).standard_normal(pm.ncols)
        rt, uct = torch.from_numpy(r).cuda(), torch.from_numpy(uc).cuda()
        y = torch.empty(pm.ncols, dtype=torch.float64, device="cuda")
        _lib.check(lib.smg_spmv_transpose(op.handle, D.ptr(rt), D.ptr(y), D.stream_handle()))
        ok_r = bool(np.array_equal(y.cpu().numpy(), O.spmv_transpose(pm, r)))
        _lib.check(lib.smg_prolong_add(op.handle, D.ptr(uct), D.ptr(rt), D.stream_handle()))
        ref = r.copy()
        ref += O.spmv(pm, uc)
        transfers.append({"level": l, "restrict_bitwise": ok_r,
                          "prolong_add_bitwise": bool(np.array_equal(rt.cpu().numpy(), ref))})
    out["transfers"] = transfers
    u = ur.copy()
    P.vcycle(h, b, u)
    ref = O.vcycle(h, b, ur.copy())
    out["vcycle_rel_diff"] = float(np.linalg.norm(u - ref) / np.linalg.norm(ref))
    t0 = time.perf_counter()
    _, hg = P.solve_stationary(h, b, u0, 1e-10, args.max_cycles)
    out["gpu_solve_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, ho = O.solve_stationary(h, b, u0, 1e-10, args.max_cycles)
    out["cpu_oracle_solve_s"] = time.perf_counter() - t0
    out["cycles_gpu"] = len(hg) - 1
    out["cycles_oracle"] = len(ho) - 1
    out["history_max_rel_diff"] = float(np.max(np.abs(np.array(hg) / np.array(ho) - 1.0)))
    out["final_rel_residual"] = hg[-1]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
