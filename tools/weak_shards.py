import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1602_07106_b200 import _lib, hashing
L = _lib.load()
for N in (1, 2, 4, 8):
    p = hashing.c_params(hashing.HashConfig(), n=N * 10**8, d=10)
    out = torch.empty(2 * 10**9, dtype=torch.int64, device="cuda")
    prb = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    res = []
    for r in range(N):
        lo = r * 10**9
        f = lambda: _lib.check(L.parba_generate(p, lo, lo + 10**9, out.data_ptr(), prb.data_ptr(), st))
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): f()
        e1.record(); torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 3)
    print(N, " ".join(f"{x:.2f}" for x in res), "ms; max", f"{max(res):.2f}")
    del out
