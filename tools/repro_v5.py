"""Isolate a failing SpMV epilogue under SMG_SPMV_VARIANT (one op per process)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tests.golden import fixtures
from paper_2402_12947_b200 import _lib, device as D

op_name = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else "c1s"
z, h = fixtures.load(name)
lib = _lib.load()
lv = h.levels[0]
A = D.device_operator(lv.a)
P = D.device_operator(lv.prolongation.matrix, with_transpose=True)
b = torch.from_numpy(z["g/b"]).cuda()
u = torch.from_numpy(z["g/u_rand"]).cuda()
y = torch.empty_like(u)
d = torch.zeros_like(u)
sh = torch.cuda.current_stream().cuda_stream
if op_name == "spmv":
    _lib.check(lib.smg_spmv(A.handle, D.ptr(u), D.ptr(y), sh))
elif op_name == "residual":
    _lib.check(lib.smg_residual(A.handle, D.ptr(b), D.ptr(u), D.ptr(y), sh))
elif op_name == "jacobi":
    _lib.check(lib.smg_smoother_step(A.handle, D.ptr(b), D.ptr(u), D.ptr(y), D.ptr(d), 0, 1.5, 0., 0., sh))
elif op_name == "chebnext":
    _lib.check(lib.smg_smoother_step(A.handle, D.ptr(b), D.ptr(u), D.ptr(y), D.ptr(d), 2, 1.5, .3, .7, sh))
elif op_name == "restrict":
    yc = torch.empty(P.ncols, dtype=torch.float64, device="cuda")
    _lib.check(lib.smg_spmv_transpose(P.handle, D.ptr(u), D.ptr(yc), sh))
elif op_name == "prolong":
    uc = torch.from_numpy(z["g/uc"]).cuda()
    _lib.check(lib.smg_prolong_add(P.handle, D.ptr(uc), D.ptr(u), sh))
torch.cuda.synchronize()
print(op_name, "ok")
