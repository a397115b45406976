"""Per-shard device times of the bench workloads for N = 1, 2, 4, 8 ranks,
measured one shard after another on ONE GPU (the pool has one GPU per
lease).  Each rank's shard is the contiguous edge-ID range bench.py gives it
(parallel.shard_range) and runs the same entry points (parba_generate /
count_shard_device).  The max over shards is the step time the N-GPU run
would see before its collective; the NCCL reduce (800 KB window, 400 MB full
histogram) is not in these numbers.  This is a balance check of the
partition, not a multi-GPU measurement.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1602_07106_b200 as pb
from paper_1602_07106_b200 import _lib

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
L = _lib.load()


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {"note": "per-shard device ms measured sequentially on one B200; max = projected N-GPU step before the "
               "NCCL reduce; eff = T(N=1) / (N * max); 'balanced' = the counting modes' shards re-cut to equal "
               "cost from the equal-shard times (parallel.balanced_cuts, as bench.py does at N > 1)"}
modes = [("store_c2", dict(n=10**8, d=10), None, 5), ("window_c3", dict(n=10**9, d=100), 10**5, 1),
         ("full_c4", dict(n=10**8, d=16), 10**8, 3), ("window_c5", dict(n=10**10, d=100), 10**5, 1)]
only = sys.argv[1:]
for name, kw, K, reps in modes:
    if only and name not in only:
        continue
    p = pb.GenParams(**kw)
    out = None
    if K is None:
        out = torch.empty((p.m, 2), dtype=torch.int64, device=dev)
    prb = torch.zeros(1, dtype=torch.int64, device=dev)
    cp = p._device_params(dev)
    rows = {}
    t1 = None
    for N in (1, 2, 4, 8):
        ms = []
        for r in range(N):
            lo, hi = pb.parallel.shard_range(0, p.m, r, N)
            if K is None:
                f = lambda: _lib.check(L.parba_generate(cp, lo, hi, out.data_ptr(), prb.data_ptr(), st.cuda_stream))
            else:
                counts = torch.zeros(K, dtype=torch.int32 if K == p.n else torch.int64, device=dev)
                f = lambda: pb.parallel.count_shard_device(p, K, lo, hi, counts=counts, probes=prb, device=dev)
            ms.append(timed(f, reps))
        t1 = t1 if t1 is not None else ms[0]
        rows[N] = {"shard_ms": [round(x, 3) for x in ms], "max_ms": round(max(ms), 3),
                   "edges_per_s_projected": p.m / max(ms) * 1e3, "eff": t1 / (N * max(ms))}
        if K is not None and N > 1:  # the bench's counting modes: cuts re-balanced by the measured step
            cuts = pb.parallel.balanced_cuts([pb.parallel.shard_range(0, p.m, r, N)[0] for r in range(N)] + [p.m], ms)
            bms = []
            for r in range(N):
                lo, hi = cuts[r], cuts[r + 1]
                counts = torch.zeros(K, dtype=torch.int32 if K == p.n else torch.int64, device=dev)
                f = lambda: pb.parallel.count_shard_device(p, K, lo, hi, counts=counts, probes=prb, device=dev)
                bms.append(timed(f, reps))
            rows[N]["balanced"] = {"shard_ms": [round(x, 3) for x in bms], "max_ms": round(max(bms), 3),
                                   "eff": t1 / (N * max(bms))}
        print(name, N, rows[N], flush=True)
    res[name] = rows
    del out
    torch.cuda.empty_cache()
print(json.dumps(res))
