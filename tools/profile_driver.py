"""Deterministic kernel sequence for ncu captures (C2 unless --workload).

    python tools/profile_driver.py            # plain run (must exit 0 before ncu)
    ncu --nvtx --nvtx-include "sweeps/" -k regex:csr_tile ... python tools/profile_driver.py

Launch order after setup (every call goes through the C-ABI), each phase in
an NVTX range so ncu can select it (`--nvtx --nvtx-include "<range>/"`):
  warm      WARM V-cycles (graph replays),
  vcycle    one more V-cycle (the launch list reads this one),
  sweeps    one ChebNext (or Jacobi) step per non-coarse level, finest first,
  lc        one fused local correction per level that has one.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

WARM = 2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    args = ap.parse_args()
    import torch
    from paper_2402_12947_b200 import _lib, configs, device as D
    from paper_2402_12947_b200.smoothers import SmootherConfig
    from paper_2402_12947_b200.mg import DeviceHierarchy
    h, b_host, _ = configs.build(configs.WORKLOADS[args.workload])
    dh = DeviceHierarchy(h.levels, h.coarse_factor)
    lib = _lib.load()
    sh = D.stream_handle()
    b = torch.from_numpy(b_host).cuda()
    u = torch.zeros_like(b)
    dh.vcycle(b, u)   # captures the V-cycle graph, then replays it
    torch.cuda.synchronize()
    per = dh.launches_per_vcycle()
    nvtx = torch.cuda.nvtx
    nvtx.range_push("warm")
    for _ in range(WARM):
        dh.vcycle(b, u)
    torch.cuda.synchronize()
    nvtx.range_pop()
    offsets = {"launches_per_vcycle": per}
    nvtx.range_push("vcycle")
    dh.vcycle(b, u)
    torch.cuda.synchronize()
    nvtx.range_pop()
    k = 0
    offsets["sweeps"] = []
    nvtx.range_push("sweeps")
    for li, lv in enumerate(h.levels[:-1]):
        op = dh.ops[li]
        cfg = lv.smoother
        n = op.nrows
        xa = torch.randn(n, dtype=torch.float64, device="cuda")
        xb = torch.empty_like(xa)
        d = torch.zeros_like(xa)
        bl = torch.randn(n, dtype=torch.float64, device="cuda")
        lam, frac = SmootherConfig.from_any(cfg).chebyshev_parameters()
        theta = 0.5 * (lam + frac * lam)
        kind = 2 if frac < 1.0 else 0   # ChebNext, or the Jacobi step
        _lib.check(lib.smg_smoother_step(op.handle, D.ptr(bl), D.ptr(xa), D.ptr(xb), D.ptr(d),
                                         kind, theta, 0.3, 0.7, sh))
        offsets["sweeps"].append({"level": li, "launch": k, "rows": n, "nnz": op.nnz,
                                  "step": kind})
        k += 1
    torch.cuda.synchronize()
    nvtx.range_pop()
    k = 0
    offsets["lc"] = []
    nvtx.range_push("lc")
    for li, corr in enumerate(dh.corrs):
        if corr is None:
            continue
        n = dh.ops[li].nrows
        bl = torch.randn(n, dtype=torch.float64, device="cuda")
        ul = torch.randn(n, dtype=torch.float64, device="cuda")
        _lib.check(lib.smg_local_correct(corr.handle, D.ptr(bl), D.ptr(ul), sh))
        offsets["lc"].append({"level": li, "launch": k})
        k += 1
    torch.cuda.synchronize()
    nvtx.range_pop()
    print(json.dumps(offsets))


if __name__ == "__main__":
    main()
