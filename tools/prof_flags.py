"""One option-flag generation call for an ncu launch list:
python tools/prof_flags.py npe|nsl|both  (n=1e7, d=10, K12 seed, all edges)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1602_07106_b200 as pb

kind = sys.argv[1] if len(sys.argv) > 1 else "npe"
kw = {"npe": dict(no_parallel_edges=True), "nsl": dict(no_self_loops=True),
      "both": dict(no_self_loops=True, no_parallel_edges=True)}[kind]
k = 12
seed = np.array([x for a in range(k) for b in range(a + 1, k) for x in (a, b)], dtype=np.uint64)
p = pb.GenParams(n=10**7, d=10, n0=k, seed_edges=seed, **kw)
out = torch.empty((p.m - p.m0, 2), dtype=torch.int64, device="cuda")
for _ in range(2):
    pb.generate_block_device(p.m0, p.m, p, out=out)
torch.cuda.synchronize()
print("ok")
