"""Apply a LocalCorrection with the given patch sizes on cuda:0 and compare with the oracle."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import scipy.linalg as sl
from paper_2402_12947_b200.smoothers import LocalCorrection
from paper_2402_12947_b200.sparse import DenseFactor
import paper_2402_12947_b200 as P
from oracle import oracle as O

sizes = [int(s) for s in sys.argv[1].split(",")]
rng = np.random.default_rng(0)
n = sum(sizes) + 100
perm = rng.permutation(n)
regs, st = [], 0
for nd in sizes:
    idx = np.sort(perm[st:st + nd]); st += nd
    dec = float(os.environ.get("COND_DECADES", "0"))
    if dec > 0:
        q, _ = np.linalg.qr(rng.standard_normal((nd, nd)))
        a = (q * np.logspace(0, -dec, nd)) @ q.T
        a = 0.5 * (a + a.T)
    else:
        m = rng.standard_normal((nd, nd)); a = m @ m.T + nd * np.eye(nd)
    c = sl.cholesky(a, lower=True)
    regs.append((idx, DenseFactor("cholesky", (c, True), nd)))
lc = LocalCorrection(tuple(regs), n)
r = rng.standard_normal(n)
out = P.apply_local_correction(lc, r)
torch.cuda.synchronize()
ref = O.apply_local_correction(lc, r)
print(sys.argv[1][:60], "rel", np.linalg.norm(out - ref) / np.linalg.norm(ref))
