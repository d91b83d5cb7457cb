"""Per-phase SM cycles of the symmetric-inverse patch path (thread 0 of each
CTA; -DSMG_PATCH_TRACE build): chunk bookkeeping, ring wait, row part, column
part, barrier, refill issue, per region size.  Diagnostic only.

    python tools/build_variant.py trace -DSMG_PATCH_TRACE      # here
    python tools/trace_sym.py                                   # on the GPU box
"""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SMG_LIB"] = os.path.join(ROOT, "paper_2402_12947_b200", "lib", "libsimplexmg_b200_trace.so")


def main():
    import torch
    from paper_2402_12947_b200 import _lib, device as D
    from paper_2402_12947_b200.sparse import CsrMatrix
    from tools.c5_patch_sweep import make
    lib = _lib.load()
    lib.smg_debug_patch_trace.argtypes = [ctypes.c_void_p]
    n = 600_000
    op = D.DeviceOperator(CsrMatrix.identity(n))
    r = torch.randn(n, dtype=torch.float64, device="cuda")
    o = torch.empty_like(r)
    names = ["unused", "ring_wait", "blocks", "butterfly", "barrier", "issue_combine", "chunks"]
    for sizes in ([512], [256], [192], [512] * 296, [512] * 1000):
        lc = make(np.array(sizes), n)
        dc = D.DeviceCorrection(op, lc)
        for _ in range(3):
            _lib.check(lib.smg_apply_local_correction(dc.handle, D.ptr(r), D.ptr(o), D.stream_handle()))
        torch.cuda.synchronize()
        zero = np.zeros((256, 16), dtype=np.uint64)
        # counters accumulate: read before and after one application
        before = np.zeros((256, 16), dtype=np.uint64)
        assert lib.smg_debug_patch_trace(before.ctypes.data) == 0
        _lib.check(lib.smg_apply_local_correction(dc.handle, D.ptr(r), D.ptr(o), D.stream_handle()))
        torch.cuda.synchronize()
        after = np.zeros((256, 16), dtype=np.uint64)
        assert lib.smg_debug_patch_trace(after.ctypes.data) == 0
        k = min(256, len(sizes))
        acc = (after[:k, 8:15].astype(np.int64) - before[:k, 8:15].astype(np.int64)).mean(axis=0)
        tot = (after[:k, 6].astype(np.int64) - after[:k, 0].astype(np.int64)).mean()
        print(json.dumps({"sizes": f"{sizes[0]} x{len(sizes)}", "total_cycles": float(tot),
                          **{nm: float(v) for nm, v in zip(names, acc)}}), flush=True)
        del dc


if __name__ == "__main__":
    main()
