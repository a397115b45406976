"""Time the store-targets kernel (parba_generate_targets, edge-order u32
targets) on the batches of C4 (n=1e8, d=16: [0, 2^29), [2^29, 2^30),
[2^30, 1.6e9)) against the partitioned count's targets pass of the same
batches (ncu launch list: 2.49 / 2.76 / 2.76 ms).  CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1602_07106_b200 as pb

p = pb.GenParams(n=10**8, d=16)
dev = torch.device("cuda", 0)
L = pb._lib.load()
cp = p._device_params(dev)
t = torch.empty(1 << 29, dtype=torch.int32, device=dev)
prb = torch.zeros(1, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream(dev).cuda_stream
for lo, hi in ((0, 1 << 29), (1 << 29, 1 << 30), (1 << 30, p.m)):
    f = lambda: pb._lib.check(L.parba_generate_targets(cp, lo, hi, t.data_ptr(), prb.data_ptr(), st))
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"[{lo}, {hi}): {ms:.3f} ms = {(hi - lo) / ms / 1e6:.3e} edges/s")
