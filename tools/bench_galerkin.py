"""Time the device Galerkin product (smg_galerkin) against the reference's host
scipy product, level by level, and check they are bit-identical.

    python tools/bench_galerkin.py [C2|C3|C4 ...] [--reps 3] [--out FILE]

Per level: `gpu_ms` = smg_galerkin alone (operators already on the device,
result left on the device; median of reps), `gpu_to_host_ms` adds the copy of
the result into host CSR arrays, `cpu_ms` = scipy ``ps.T @ (a @ ps)``
(sparse.py:147-154, one run), `bitwise` = identical arrays.  The algorithmic
traffic figure counts reading A, P (twice: P and CSR(P^T)) and AP once and
writing AP and A_c once (12 B per nonzero, 8 B per row offset).
"""

import ctypes
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = 3
    out = None
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
        args = [a for a in args if a != str(reps)]
    if "--out" in sys.argv:
        out = sys.argv[sys.argv.index("--out") + 1]
        args = [a for a in args if a != out]
    names = args or ["C2"]
    import torch
    from paper_2402_12947_b200 import _lib, configs
    from paper_2402_12947_b200 import device as D
    from paper_2402_12947_b200.sparse import host_triple_product
    lib = _lib.load()
    records = []
    for name in names:
        wl = getattr(configs, name)
        t0 = time.perf_counter()
        h = configs.build(wl)[0]
        setup_s = time.perf_counter() - t0
        print(json.dumps({"workload": wl.name, "setup_s": setup_s,
                          "setup_times": getattr(h, "setup_times", None)}), flush=True)
        records.append({"workload": wl.name, "setup_s": setup_s,
                        "setup_times": getattr(h, "setup_times", None)})
        for l in range(len(h.levels) - 1):
            a, p = h.levels[l].a, h.levels[l].prolongation.matrix
            oa, op = D.device_operator(a), D.device_operator(p, with_transpose=True)
            torch.cuda.synchronize()
            times = []
            res = None
            for _ in range(reps + 1):
                hd = ctypes.c_void_p()
                t0 = time.perf_counter()
                _lib.check(lib.smg_galerkin(oa.handle, op.handle, ctypes.byref(hd), None))
                torch.cuda.synchronize()
                times.append(time.perf_counter() - t0)
                if res is None:
                    t1 = time.perf_counter()
                    res = D._csr_result_to_host(lib, hd)
                    copy_s = time.perf_counter() - t1
                else:
                    lib.smg_csr_destroy(hd)
            gpu_s = float(np.median(times[1:]))
            t0 = time.perf_counter()
            ref = host_triple_product(p, a)
            cpu_s = time.perf_counter() - t0
            _, _, ptr, col, val = res
            same = (np.array_equal(ptr, ref.row_offsets) and np.array_equal(col, ref.col_indices)
                    and np.array_equal(val, ref.values))
            # A P nnz (for the traffic figure): rows of P^T (A P) before the second product
            nnz_ap = int(D.matmul(a, p)[2][-1])
            traffic = (12 * a.nnz + 8 * a.nrows + 2 * (12 * p.nnz + 8 * p.nrows) +
                       2 * (12 * nnz_ap + 8 * a.nrows) + 12 * ref.nnz + 8 * ref.nrows)
            rec = {"workload": wl.name, "level": l + 1, "fine_rows": a.nrows, "fine_nnz": a.nnz,
                   "p_nnz": p.nnz, "ap_nnz": nnz_ap, "coarse_rows": ref.nrows,
                   "coarse_nnz": ref.nnz, "gpu_ms": gpu_s * 1e3,
                   "gpu_to_host_ms": (gpu_s + copy_s) * 1e3, "cpu_ms": cpu_s * 1e3,
                   "speedup": cpu_s / gpu_s, "bitwise": bool(same),
                   "traffic_gb_s": traffic / gpu_s / 1e9, "setup_s": setup_s}
            records.append(rec)
            print(json.dumps(rec), flush=True)
    if out:
        with open(out, "w") as f:
            json.dump(records, f, indent=1)


if __name__ == "__main__":
    main()
