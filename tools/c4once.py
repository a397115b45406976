import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1602_07106_b200 as pb
from paper_1602_07106_b200 import _lib
dev = torch.device("cuda", 0); st = torch.cuda.current_stream(dev).cuda_stream
L = _lib.load(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1] else _lib.load()
p = pb.GenParams(n=10**8, d=16); cp = p._device_params(dev)
prb = torch.zeros(1, dtype=torch.int64, device=dev); c = torch.zeros(p.n, dtype=torch.int32, device=dev)
for _ in range(2):
    _lib.check(L.parba_degree_full(cp, 0, p.m, c.data_ptr(), prb.data_ptr(), st))
torch.cuda.synchronize()
