"""One full C4 launch (n=1e8, d=16, all 1.6e9 edges, u32 counts) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1602_07106_b200 as pb

dev = torch.device("cuda", 0)
L = pb._lib.load()
st = torch.cuda.current_stream(dev).cuda_stream
p = pb.GenParams(n=10**8, d=16)
c = torch.zeros(p.n, dtype=torch.int32, device=dev)
prb = torch.zeros(1, dtype=torch.int64, device=dev)
for _ in range(2):
    pb._lib.check(L.parba_degree_full(p._device_params(dev), 0, p.m, c.data_ptr(), prb.data_ptr(), st))
torch.cuda.synchronize()
print("ok")
