"""no_self_loops on a degree sequence (power-law, zeros included, n=1e7):
store-mode edges/s of the node kernel path.  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1602_07106_b200 as pb

rng = np.random.default_rng(3)
n = 10**7
deg = np.minimum(rng.zipf(2.2, size=n) + 4, 1000).astype(np.uint64)
deg[::20] = 0
k = 12
seed = np.array([x for a in range(k) for b in range(a + 1, k) for x in (a, b)], dtype=np.uint64)
p = pb.GenParams(n=k + n, n0=k, degrees=deg, seed_edges=seed, no_self_loops=True)
out = torch.empty((p.m - p.m0, 2), dtype=torch.int64, device="cuda")
pb.generate_block_device(p.m0, p.m, p, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    pb.generate_block_device(p.m0, p.m, p, out=out)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 3e3
print(json.dumps({"m": p.m - p.m0, "ms": t * 1e3, "edges_per_s": (p.m - p.m0) / t}))
