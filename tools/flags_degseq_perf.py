"""no_parallel_edges on a power-law degree sequence (hubs up to 1e4 edges):
the node kernel's worst case.  python tools/flags_degseq_perf.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1602_07106_b200 as pb

rng = np.random.default_rng(0)
n = 10**6
for cap in (100, 1000, 10_000):
    deg = np.sort(np.minimum(rng.zipf(2.0, size=n) + 2, cap)).astype(np.uint64)  # hubs late: feasible pools
    seed = np.array([x for u in range(64) for v in range(u + 1, 64) for x in (u, v)], dtype=np.uint64)
    p = pb.GenParams(n=64 + n, n0=64, degrees=deg, seed_edges=seed, no_parallel_edges=True)
    out = torch.empty((p.m - p.m0, 2), dtype=torch.int64, device="cuda")
    pb.generate_block_device(p.m0, p.m, p, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pb.generate_block_device(p.m0, p.m, p, out=out)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"cap {cap}: m={p.m - p.m0} max deg {int(deg.max())}: {(p.m - p.m0) / dt:.3e} edges/s ({dt*1e3:.1f} ms)", flush=True)
