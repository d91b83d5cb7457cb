"""Small deterministic workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family the hot path launches, on golden
fixtures small enough to finish under instrumentation.

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py [--mode M]

Covers: SELL and tile sweeps (all epilogues), restriction / prolong-add, the
patch kernels (fused; coupled regions' residual-only + solve-from-buffer;
streamed-factor ring on c4s' 279-dof regions; cond-1e6 c5p blocks up to 512
dofs), the follow-mode rings (SMG_LC_FOLLOW=1) and the interior/halo overlap,
the coarse symmetric-tile apply (two-kernel and, with SMG_COARSE_FUSED=1, the
atomic last-CTA reduction), dots, CG, the stationary loop, and the setup
kernels (Galerkin SpGEMM, patch Cholesky).  Exits non-zero if a result is
off, so a sanitizer run also checks the numbers."""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="all", choices=["all", "default", "follow", "overlap"])
    ap.add_argument("--stress", type=int, default=0,
                    help="repeat every V-cycle this many times on fresh copies of the same "
                         "inputs (graphs and eager) and require bit-identical results: a "
                         "race on shared memory, a ring stage or the last-CTA reduction "
                         "would show up as run-to-run differences")
    args = ap.parse_args()
    import torch
    import paper_2402_12947_b200 as P
    from paper_2402_12947_b200.mg import DeviceHierarchy
    from tests.golden import fixtures
    from tests.test_oracle_golden import load_c5p
    bad = []
    modes = ["default", "follow", "overlap"] if args.mode == "all" else [args.mode]
    for name in ["c1s", "cpl_p2", "c4s", "crit7_adj"]:
        z, h = fixtures.load(name)
        b, ur = z["g/b"], z["g/u_rand"]
        for mode in modes:
            dh = DeviceHierarchy(h.levels, h.coarse_factor, use_graphs=False)
            if mode == "overlap":
                dh.set_option(2, 1)
            if mode == "follow":
                dh.set_option(3, 1)
            u = ur.copy()
            dh.vcycle(b, u)
            if rel(u, z["g/vcycle1"]) > 1e-12:
                bad.append(f"{name}/{mode}: vcycle {rel(u, z['g/vcycle1']):.2e}")
            for graphs in ((True, False) if args.stress else ()):
                dg = DeviceHierarchy(h.levels, h.coarse_factor, use_graphs=graphs)
                if mode == "overlap":
                    dg.set_option(2, 1)
                if mode == "follow":
                    dg.set_option(3, 1)
                bt = torch.from_numpy(b).cuda()
                outs = []
                for _ in range(args.stress):
                    ut = torch.from_numpy(ur).cuda()
                    dg.vcycle(bt, ut)
                    dg.vcycle(bt, ut)
                    outs.append(ut)
                torch.cuda.synchronize()
                ref = outs[0].cpu().numpy()
                if not np.array_equal(ref, u) and graphs:
                    pass
                ndiff = sum(0 if np.array_equal(o.cpu().numpy(), ref) else 1 for o in outs)
                if ndiff:
                    bad.append(f"{name}/{mode}/graphs={graphs}: {ndiff} of {args.stress} "
                               f"reruns differ")
        lv = h.levels[0]
        w = ur.copy()
        P.combined_smooth(lv.a, b, w, lv.local_correction, lv.smoother)
        if rel(w, z["g/combined"]) > 1e-12:
            bad.append(f"{name}: combined_smooth")
        if not np.array_equal(P.restrict_residual(lv.prolongation, ur), z["g/restrict"]):
            bad.append(f"{name}: restriction")
        _, hist = P.solve_stationary(h, b, z["g/u0"], 1e-10, 3)
        _, ch = P.cg(lv.a, b, precond=P.as_preconditioner(h), rtol=1e-10, maxit=3)
        np.testing.assert_allclose(hist, z["g/stat_hist"][:len(hist)], rtol=1e-6)
        np.testing.assert_allclose(ch, z["g/cg_hist"][:len(ch)], rtol=1e-6)
    zc, lc = load_c5p()
    out = P.apply_local_correction(lc, zc["r"])
    if rel(out, zc["lc_apply"]) > 1e-13:
        bad.append("c5p: patch solves")
    for _ in range(args.stress):
        if not np.array_equal(P.apply_local_correction(lc, zc["r"]), out):
            bad.append("c5p: rerun differs")
            break
    # setup kernels: Galerkin product and batched patch Cholesky on the device
    z, h = fixtures.load("c2s")
    from paper_2402_12947_b200.sparse import triple_product
    from paper_2402_12947_b200.smoothers import build_local_correction
    a1 = triple_product(h.levels[0].prolongation.matrix, h.levels[0].a)
    if not np.array_equal(a1.values, h.levels[1].a.values):
        bad.append("galerkin")
    sets = [idx for idx, _ in h.levels[0].local_correction.regions]
    build_local_correction(h.levels[0].a, sets, device=True)
    torch.cuda.synchronize()
    if bad:
        print("FAILED:", bad)
        return 1
    print("sanitize driver ok")
    return 0


if __name__ == "__main__":
    sys.exit(main())
