"""Degree counts with K = n when 2m >= 2^32 (u64 window over all nodes):
n=1e9, d=10, edge range of 2e9 at the top of the ID space.  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1602_07106_b200 as pb

dev = torch.device("cuda", 0)
res = {}
for name, n, d, span in (("n1e9_d10", 10**9, 10, 2 * 10**9), ("n4e8_d16", 4 * 10**8, 16, 2 * 10**9)):
    p = pb.GenParams(n=n, d=d)
    lo, hi = p.m - span, p.m
    counts = torch.zeros(n, dtype=torch.int64, device=dev)
    prb = torch.zeros(1, dtype=torch.int64, device=dev)
    pb.parallel.count_shard_device(p, n, lo, hi, counts=counts, probes=prb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        pb.parallel.count_shard_device(p, n, lo, hi, counts=counts, probes=prb)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3e3
    res[name] = {"edges": span, "ms": t * 1e3, "edges_per_s": span / t, "dtype": str(counts.dtype)}
    del counts
print(json.dumps(res))
