"""Phase breakdown of the batched patch solve (SM clock cycles per CTA).

    python tools/trace_patch.py build          # here: builds lib/libsimplexmg_b200_trace.so
    python tools/trace_patch.py run c3s c2s c5 # on the GPU box

The trace build compiles patch_kernels.cu with -DSMG_PATCH_TRACE: thread 0 of
the first 256 CTAs stamps clock64() at kernel start (0), after the dependency
wait (1), residual done (2), factor staged (3), forward solve done (4),
backward solve done (5) and scatter done (6).  Diagnostic only.
"""

import ctypes
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_12947_b200 import build_lib  # noqa: E402

TRACE_LIB = os.path.join(build_lib.LIBDIR, "libsimplexmg_b200_trace.so")
PHASES = ["pdl_wait", "residual", "factor_wait", "forward", "backward", "scatter"]


def build():
    flags = [f for f in build_lib.FLAGS if f not in ("-Xptxas", "-v")]
    cmd = [build_lib.NVCC] + flags + ["-DSMG_PATCH_TRACE", "-o", TRACE_LIB] + build_lib.sources()
    subprocess.run(cmd, check=True, capture_output=True)
    print(TRACE_LIB)


def load_trace_lib():
    from paper_2402_12947_b200 import _lib
    lib = ctypes.CDLL(TRACE_LIB)
    for name, (res, args) in _lib.PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    lib.smg_debug_patch_trace.argtypes = [ctypes.c_void_p]
    _lib._lib = lib
    return lib


def trace(lib, lc_host, a_host, label, apply=False):
    import torch
    from paper_2402_12947_b200 import device as D, _lib
    op = D.device_operator(a_host)
    dc = D.DeviceCorrection(op, lc_host)
    n = a_host.nrows
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    u = torch.randn(n, dtype=torch.float64, device="cuda")
    for _ in range(5):
        if apply:  # r -> S_c r (the C5 micro-benchmark's call)
            _lib.check(lib.smg_apply_local_correction(dc.handle, D.ptr(b), D.ptr(u),
                                                      D.stream_handle()))
        else:
            _lib.check(lib.smg_local_correct(dc.handle, D.ptr(b), D.ptr(u), D.stream_handle()))
    torch.cuda.synchronize()
    buf = np.zeros((256, 8), dtype=np.uint64)
    assert lib.smg_debug_patch_trace(buf.ctypes.data) == 0
    nreg = min(256, len(lc_host.regions))
    t = buf[:nreg].astype(np.int64)
    d = np.diff(t[:, :7], axis=1)
    sizes = [len(lc_host.regions[k][0]) for k in range(nreg)]
    return {"label": label, "regions": len(lc_host.regions), "dofs_mean": float(np.mean(sizes)),
            "cycles_mean": {p: float(d[:, i].mean()) for i, p in enumerate(PHASES)},
            "cycles_max": {p: int(d[:, i].max()) for i, p in enumerate(PHASES)},
            "total_mean": float((t[:, 6] - t[:, 0]).mean())}


def run(names):
    lib = load_trace_lib()
    out = []
    for name in names:
        if name == "c5":
            import bench
            from paper_2402_12947_b200 import stencil
            a = stencil.p2_tet_laplacian(63)
            lc = bench.make_c5_patches(a.nrows)
            out.append(trace(lib, lc, a, "c5 grid 63 (apply; phase 3->4 forward, 4->5 backward)",
                             apply=True))
        else:
            from tests.golden import fixtures
            z, h = fixtures.load(name)
            lv = h.levels[0]
            out.append(trace(lib, lv.local_correction, lv.a, name))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(sys.argv[2:])
