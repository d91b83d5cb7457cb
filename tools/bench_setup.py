"""Time the device prolongation construction (smg_prolongation_build) against
the host restatement of transfer.py:117-150, level by level, and check they
are bit-identical.

    python tools/bench_setup.py [C2|C3|C4 ...] [--out FILE]

Per level: `gpu_ms` = device build_prolongation (host bin index + inverse
Jacobians + upload + kernel + copy back), `kernel_free_ms` = the host part of
it alone (CellLocator construction), `cpu_ms` = the vectorised host version,
`bitwise` = identical CSR arrays.
"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    names = [a for a in sys.argv[1:] if not a.startswith("--")]
    out = None
    if "--out" in sys.argv:
        out = sys.argv[sys.argv.index("--out") + 1]
        names = [a for a in names if a != out]
    names = names or ["C2"]
    import torch
    from paper_2402_12947_b200 import configs
    from paper_2402_12947_b200.fem import build_dofmap
    from paper_2402_12947_b200.transfer import CellLocator, build_prolongation
    records = []
    for name in names:
        w = getattr(configs, name)
        meshes = configs.build_meshes(w)
        dms = [build_dofmap(m, w.degree) for m in meshes]
        from paper_2402_12947_b200.fem import assemble_poisson
        assemble_poisson(meshes[-1], dms[-1], device=True)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sd = assemble_poisson(meshes[0], dms[0], device=True)
        gpu_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        sh = assemble_poisson(meshes[0], dms[0], device=False)
        cpu_s = time.perf_counter() - t0
        same_pat = (np.array_equal(sd.a.row_offsets, sh.a.row_offsets)
                    and np.array_equal(sd.a.col_indices, sh.a.col_indices))
        rel = float(np.max(np.abs(sd.a.values - sh.a.values)) / np.max(np.abs(sh.a.values)))
        rec = {"workload": w.name, "step": "assembly", "dofs": sd.a.nrows, "nnz": sd.a.nnz,
               "cells": int(meshes[0].n_cells), "gpu_ms": gpu_s * 1e3, "cpu_ms": cpu_s * 1e3,
               "speedup": cpu_s / gpu_s, "same_pattern": bool(same_pat), "max_rel_diff": rel}
        records.append(rec)
        print(json.dumps(rec), flush=True)
        del sh
        for l in range(len(meshes) - 1):
            build_prolongation(dms[l], meshes[l + 1], dms[l + 1], device=True)  # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            p_dev = build_prolongation(dms[l], meshes[l + 1], dms[l + 1], device=True)
            gpu_s = time.perf_counter() - t0
            t0 = time.perf_counter()
            CellLocator(meshes[l + 1])
            loc_s = time.perf_counter() - t0
            t0 = time.perf_counter()
            p_host = build_prolongation(dms[l], meshes[l + 1], dms[l + 1], device=False)
            cpu_s = time.perf_counter() - t0
            same = (np.array_equal(p_dev.row_offsets, p_host.row_offsets)
                    and np.array_equal(p_dev.col_indices, p_host.col_indices)
                    and np.array_equal(p_dev.values, p_host.values))
            rec = {"workload": w.name, "fine_level": l, "fine_dofs": p_dev.nrows,
                   "coarse_dofs": p_dev.ncols, "coarse_cells": int(meshes[l + 1].n_cells),
                   "p_nnz": p_dev.nnz, "gpu_ms": gpu_s * 1e3, "host_locator_ms": loc_s * 1e3,
                   "cpu_ms": cpu_s * 1e3, "speedup": cpu_s / gpu_s, "bitwise": bool(same)}
            records.append(rec)
            print(json.dumps(rec), flush=True)
    if out:
        with open(out, "w") as f:
            json.dump(records, f, indent=1)


if __name__ == "__main__":
    main()
