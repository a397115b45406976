"""(Record of a dropped experiment: the PARBA_LOW_DIV knob is not in the shipped
library; see profiles/r02_ab_c4_scatter_lean.txt.)
A/B of the hot-low-node split of the partitioned full histogram
(PARBA_LOW_DIV = D: targets below ~K/D counted by direct L2 atomics in the
store-targets pass, the rest bucket-sorted).  C4 (n=1e8, d=16) and two other
shapes; every setting is checked element-wise against D = 0.  One JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1602_07106_b200 as pb

dev = torch.device("cuda", 0)
L = pb._lib.load()
st = torch.cuda.current_stream(dev).cuda_stream
divs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,64,32,16,8,4,2").split(",")]
res = {}
for name, kw in (("C4", dict(n=10**8, d=16)), ("n2e8_d8", dict(n=2 * 10**8, d=8)),
                 ("n5e7_d32", dict(n=5 * 10**7, d=32))):
    p = pb.GenParams(**kw)
    cp = p._device_params(dev)
    prb = torch.zeros(1, dtype=torch.int64, device=dev)
    c = torch.zeros(p.n, dtype=torch.int32, device=dev)
    ref = None
    for D in divs:
        os.environ["PARBA_LOW_DIV"] = str(D)
        c.zero_()
        pb._lib.check(L.parba_degree_full(cp, 0, p.m, c.data_ptr(), prb.data_ptr(), st))
        torch.cuda.synchronize()
        if ref is None:
            ref = c.clone()
        elif not torch.equal(ref, c):
            raise SystemExit(f"{name} D={D}: counts differ from D={divs[0]}")
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
        res[f"{name}_D{D}"] = {"ms": round(ms, 3), "edges_per_s": p.m / ms * 1e3}
        print(name, D, round(ms, 3), f"{p.m / ms * 1e3:.4e}", flush=True)
    del ref, c
os.environ.pop("PARBA_LOW_DIV", None)
print(json.dumps(res))
