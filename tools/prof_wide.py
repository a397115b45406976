"""One wide store launch (1e9 edges at positions >= 2^32: the NC=4 path)
for ncu captures.  python tools/prof_wide.py [LIB]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1602_07106_b200 import _lib, hashing

L = _lib.load(sys.argv[1]) if len(sys.argv) > 1 else _lib.load()
p = hashing.c_params(hashing.HashConfig(), n=8 * 10**8, d=10)
out = torch.empty(2 * 10**9, dtype=torch.int64, device="cuda")
prb = torch.zeros(1, dtype=torch.int64, device="cuda")
lo = 7 * 10**9
for _ in range(2):
    _lib.check(L.parba_generate(p, lo, lo + 10**9, out.data_ptr(), prb.data_ptr(),
                                torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("ok")
