"""Apply a slice [a, b) of the seeded C5 patch set; exit code 0 iff it works."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2402_12947_b200 as P
from paper_2402_12947_b200.smoothers import LocalCorrection
from oracle import oracle as O
a, b = int(sys.argv[1]), int(sys.argv[2])
nrows = 2048383
full = bench.make_c5_patches(nrows, count=b)
regs = full.regions[a:b]
mn = int(os.environ.get("MIN_SIZE", "0"))
regs = [rg for rg in regs if len(rg[0]) >= mn]
lc = LocalCorrection(tuple(regs), nrows)
r = np.random.default_rng(1).standard_normal(nrows)
out = P.apply_local_correction(lc, r)
torch.cuda.synchronize()
ref = O.apply_local_correction(lc, r)
print(a, b, [len(i) for i, _ in regs][:8], "rel", np.linalg.norm(out - ref) / np.linalg.norm(ref))
