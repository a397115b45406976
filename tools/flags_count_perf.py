"""Option-flag degree counts at C4 scale (n=1e8, d=16, K17 seed): full u32
counts and a K=1e5 window, CUDA-event timed.  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1602_07106_b200 as pb

dev = torch.device("cuda", 0)
k = 17
seed = np.array([x for a in range(k) for b in range(a + 1, k) for x in (a, b)], dtype=np.uint64)
res = {}
for flag in ("no_self_loops", "no_parallel_edges"):
    p = pb.GenParams(n=10**8, d=16, n0=k, seed_edges=seed, **{flag: True})
    for K in (p.n, 10**5):
        lo, hi = p.m0, p.m
        f = lambda: pb.parallel.count_shard_device(p, K, lo, hi)
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            f()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 2e3
        res[f"{flag}_K{K}"] = {"ms": t * 1e3, "edges_per_s": (hi - lo) / t}
print(json.dumps(res))
