"""f4 store: owner lookups by the dense map vs the rank directory, for a
degree sequence with and without zero-degree nodes (n=1e8, mean ~13,
power-law tail).  CUDA events; prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1602_07106_b200 as pb
from paper_1602_07106_b200 import generator

dev = torch.device("cuda", 0)
res = {}
for zeros in (0.0, 0.05):
    rng = np.random.default_rng(5)
    n = 10**8
    deg = np.minimum(rng.zipf(2.0, size=n) + 7, 10_000).astype(np.uint64)
    if zeros:
        deg[rng.random(n) < zeros] = 0
    deg[0] = 10
    for dense in (True, False):
        generator.DENSE_OWNER_MAX_BYTES = (1 << 34) if dense else 0
        if dense and not zeros:  # force the map (the product skips it without zeros)
            generator.DENSE_FORCE = True
        p = pb.GenParams(n=n, degrees=deg)
        lo, hi = p.m - 10**9, p.m
        out = torch.empty((hi - lo, 2), dtype=torch.int64, device=dev)
        pb.generate_block_device(lo, hi, p, out=out, device=dev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            pb.generate_block_device(lo, hi, p, out=out, device=dev)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 3e3
        res[f"store_zeros{zeros}_{'dense' if dense else 'rank'}"] = (hi - lo) / t
        del out
        counts = torch.zeros(n, dtype=torch.int32, device=dev)
        pb.parallel.count_shard_device(p, n, lo, hi, counts=counts)
        torch.cuda.synchronize()
        e0.record()
        pb.parallel.count_shard_device(p, n, lo, hi, counts=counts)
        e1.record()
        torch.cuda.synchronize()
        res[f"full_zeros{zeros}_{'dense' if dense else 'rank'}"] = (hi - lo) / (e0.elapsed_time(e1) / 1e3)
        del counts, p
        torch.cuda.empty_cache()
print(json.dumps(res))
