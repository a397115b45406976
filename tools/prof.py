"""Small single-launch workloads for ncu (one GPU, no timing claims).

    python tools/prof.py store|window|full|all
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1602_07106_b200 as pb


def main(which: str) -> None:
    dev = torch.device("cuda", 0)
    L = pb._lib.load()
    st = torch.cuda.current_stream(dev).cuda_stream
    prb = torch.zeros(1, dtype=torch.int64, device=dev)
    if which in ("store", "all"):
        p = pb.GenParams(n=10**8, d=10)
        lo, hi = 0, 250_000_000  # a quarter of C2 (one launch)
        out = torch.empty((hi - lo, 2), dtype=torch.int64, device=dev)
        for _ in range(2):
            pb._lib.check(L.parba_generate(p._device_params(dev), lo, hi, out.data_ptr(), prb.data_ptr(), st))
        torch.cuda.synchronize()
        del out
    if which in ("window", "all"):
        p = pb.GenParams(n=10**9, d=100)
        lo, hi, K = 5 * 10**10, 5 * 10**10 + 2 * 10**9, 10**5
        c = torch.zeros(K, dtype=torch.int64, device=dev)
        for _ in range(2):
            pb._lib.check(L.parba_degree_window(p._device_params(dev), lo, hi, K, c.data_ptr(), prb.data_ptr(), st))
        torch.cuda.synchronize()
    if which in ("full", "all"):
        p = pb.GenParams(n=10**8, d=16)
        c = torch.zeros(p.n, dtype=torch.int32, device=dev)
        for _ in range(2):
            pb._lib.check(L.parba_degree_full(p._device_params(dev), 0, 400_000_000, c.data_ptr(), prb.data_ptr(), st))
        torch.cuda.synchronize()
    print("ok", which)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
