"""Partitioned full histogram for an ncu launch list: n from argv (default
1e8), d=16, all edges, two calls (PARBA_FULL_MODE=partition)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PARBA_FULL_MODE", "partition")
import torch

import paper_1602_07106_b200 as pb

dev = torch.device("cuda", 0)
L = pb._lib.load()
st = torch.cuda.current_stream(dev).cuda_stream
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
p = pb.GenParams(n=n, d=16)
c = torch.zeros(p.n, dtype=torch.int32, device=dev)
prb = torch.zeros(1, dtype=torch.int64, device=dev)
for _ in range(2):
    pb._lib.check(L.parba_degree_full(p._device_params(dev), 0, p.m, c.data_ptr(), prb.data_ptr(), st))
torch.cuda.synchronize()
print("ok")
