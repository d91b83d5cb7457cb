"""C5 patch set (bench.make_c5_patches) applied standalone; arg: patch count."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2402_12947_b200 as P
from oracle import oracle as O
count = int(sys.argv[1])
nrows = int(sys.argv[2]) if len(sys.argv) > 2 else 2048383
lc = bench.make_c5_patches(nrows, count=count)
r = np.random.default_rng(1).standard_normal(nrows)
out = P.apply_local_correction(lc, r)
torch.cuda.synchronize()
ref = O.apply_local_correction(lc, r)
print(count, nrows, "rel", np.linalg.norm(out - ref) / np.linalg.norm(ref))
