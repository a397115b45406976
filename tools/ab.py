"""A/B timing of alternative builds of libparba_b200.so (one GPU).

    python tools/ab.py lib1.so [lib2.so ...]

For each library: C2 store (1e9 edges into HBM), C3 window subrange (2e10
edges) and C4 full (1.6e9) with CUDA events; prints edges/s."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1602_07106_b200 import _lib, hashing


def run(path: str) -> dict:
    L = ctypes.CDLL(path)
    _lib._lib = None
    L = _lib.load(path)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    prb = torch.zeros(1, dtype=torch.int64, device=dev)
    res = {}

    def timeit(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1000 / reps

    p = hashing.c_params(hashing.HashConfig(), n=10**8, d=10)
    out = torch.empty(2 * 10**9, dtype=torch.int64, device=dev)
    t = timeit(lambda: _lib.check(L.parba_generate(p, 0, 10**9, out.data_ptr(), prb.data_ptr(), st.cuda_stream)), 5)
    res["store_c2"] = 1e9 / t
    del out
    p = hashing.c_params(hashing.HashConfig(), n=10**9, d=100)
    c = torch.zeros(10**5, dtype=torch.int64, device=dev)
    lo = 5 * 10**10
    t = timeit(lambda: _lib.check(L.parba_degree_window(p, lo, lo + 2 * 10**10, 10**5, c.data_ptr(), prb.data_ptr(), st.cuda_stream)), 2)
    res["window_c3"] = 2e10 / t
    p = hashing.c_params(hashing.HashConfig(), n=10**8, d=16)
    c = torch.zeros(10**8, dtype=torch.int32, device=dev)
    t = timeit(lambda: _lib.check(L.parba_degree_full(p, 0, 16 * 10**8, c.data_ptr(), prb.data_ptr(), st.cuda_stream)), 3)
    res["full_c4"] = 1.6e9 / t
    return res


if __name__ == "__main__":
    for path in sys.argv[1:]:
        r = run(path)
        print(os.path.basename(path), " ".join(f"{k}={v:.4e}" for k, v in r.items()), flush=True)
