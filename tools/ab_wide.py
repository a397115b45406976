"""A/B of store throughput across the kernel variants a graph's size selects:
1e9-edge shards at 0 (NC=2), 1e9 (NC=3) and 7e9 (NC=4) of an n=8e8, d=10
graph.  python tools/ab_wide.py LIB..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1602_07106_b200 import _lib, hashing

for path in sys.argv[1:]:
    _lib._lib = None
    L = _lib.load(path)
    p = hashing.c_params(hashing.HashConfig(), n=8 * 10**8, d=10)
    out = torch.empty(2 * 10**9, dtype=torch.int64, device="cuda")
    prb = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    res = []
    for lo in (0, 10**9, 7 * 10**9):
        f = lambda: _lib.check(L.parba_generate(p, lo, lo + 10**9, out.data_ptr(), prb.data_ptr(), st))
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            f()
        e1.record()
        torch.cuda.synchronize()
        res.append(1e9 / (e0.elapsed_time(e1) / 3 / 1000))
    print(os.path.basename(path), " ".join(f"{x:.3e}" for x in res), flush=True)
    del out
