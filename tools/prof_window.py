"""One C3 window launch (2e10 edges at the middle of C3) for ncu captures.
python tools/prof_window.py [LIB]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1602_07106_b200 import _lib, hashing

L = _lib.load(sys.argv[1]) if len(sys.argv) > 1 else _lib.load()
p = hashing.c_params(hashing.HashConfig(), n=10**9, d=100)
c = torch.zeros(10**5, dtype=torch.int64, device="cuda")
prb = torch.zeros(1, dtype=torch.int64, device="cuda")
lo = 5 * 10**10
for _ in range(2):
    _lib.check(L.parba_degree_window(p, lo, lo + 2 * 10**9, 10**5, c.data_ptr(), prb.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("ok")
