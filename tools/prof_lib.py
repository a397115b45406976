"""One C2 store launch of a given library build (for ncu A/B captures).
python tools/prof_lib.py LIB"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1602_07106_b200 import _lib, hashing

L = _lib.load(sys.argv[1])
p = hashing.c_params(hashing.HashConfig(), n=10**8, d=10)
out = torch.empty(2 * 10**9, dtype=torch.int64, device="cuda")
prb = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(2):
    _lib.check(L.parba_generate(p, 0, 10**9, out.data_ptr(), prb.data_ptr(), torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("ok")
