"""Full histogram (C4: n=1e8, d=16, 1.6e9 edges, u32 counts): direct atomics
vs the partitioned pass, CUDA-event timed on the launching stream, plus the
per-kernel split of the partitioned pass.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1602_07106_b200 as pb

dev = torch.device("cuda", 0)
L = pb._lib.load()
st = torch.cuda.current_stream(dev).cuda_stream
res = {}
for name, kw in (("C4", dict(n=10**8, d=16)), ("n2e7_d16", dict(n=2 * 10**7, d=16)),
                 ("n2e8_d8", dict(n=2 * 10**8, d=8))):
    p = pb.GenParams(**kw)
    ref = None
    for mode in ("direct", "partition"):
        os.environ["PARBA_FULL_MODE"] = mode
        c = torch.zeros(p.n, dtype=torch.int32, device=dev)
        prb = torch.zeros(1, dtype=torch.int64, device=dev)
        cp = p._device_params(dev)
        pb._lib.check(L.parba_degree_full(cp, 0, p.m, c.data_ptr(), prb.data_ptr(), st))
        torch.cuda.synchronize()
        if ref is None:
            ref = c.clone()
        else:
            assert torch.equal(ref, c), name
        ts = []
        for _ in range(5):
            c.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pb._lib.check(L.parba_degree_full(cp, 0, p.m, c.data_ptr(), prb.data_ptr(), st))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        res[f"{name}_{mode}"] = {"ms": round(ms, 3), "edges_per_s": p.m / ms * 1e3}
    del ref
print(json.dumps(res))
