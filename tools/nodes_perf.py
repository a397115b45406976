"""Throughput of the node-granular rows on one GPU (device-timed, CUDA events):
degree-sequence store / window / full (f4) and the option-flag node kernel
(f3).  python tools/nodes_perf.py [--n N]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1602_07106_b200 as pb
from paper_1602_07106_b200 import _lib


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1000 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10**8)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    L = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    res = {}
    rng = np.random.default_rng(0)
    n = args.n
    # f4: C2-shaped degree sequence (mean 10, power-law tail, 5% zeros)
    deg = np.minimum(rng.zipf(2.0, size=n) + 7, 10_000).astype(np.uint64)
    deg[rng.random(n) < 0.05] = 0
    deg[0] = 10
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    p = pb.GenParams(n=n, degrees=deg)
    cp = p._device_params(dev)
    t1.record()
    torch.cuda.synchronize()
    res["degseq_index_build_s"] = t0.elapsed_time(t1) / 1000
    m = p.m
    res["degseq_m"] = m
    prb = torch.zeros(1, dtype=torch.int64, device=dev)
    out = torch.empty(2 * m, dtype=torch.int64, device=dev)
    t = timeit(lambda: _lib.check(L.parba_generate(cp, 0, m, out.data_ptr(), prb.data_ptr(), st)))
    res["degseq_store_edges_per_s"] = m / t
    del out
    c = torch.zeros(10**5, dtype=torch.int64, device=dev)
    t = timeit(lambda: _lib.check(L.parba_degree_window(cp, 0, m, 10**5, c.data_ptr(), prb.data_ptr(), st)))
    res["degseq_window_edges_per_s"] = m / t
    if 2 * m < 2**32:
        c32 = torch.zeros(n, dtype=torch.int32, device=dev)
        t = timeit(lambda: _lib.check(L.parba_degree_full(cp, 0, m, c32.data_ptr(), prb.data_ptr(), st)))
        res["degseq_full_edges_per_s"] = m / t
        del c32
    # plain reference point on the same m
    q = pb.GenParams(n=n, d=10)
    cq = q._device_params(dev)
    out = torch.empty(2 * q.m, dtype=torch.int64, device=dev)
    t = timeit(lambda: _lib.check(L.parba_generate(cq, 0, q.m, out.data_ptr(), prb.data_ptr(), st)))
    res["plain_store_edges_per_s"] = q.m / t
    del out
    # f3: option flags, uniform d=10 with a K12 seed, n/10 nodes
    seed = np.array([x for u in range(12) for v in range(u + 1, 12) for x in (u, v)], dtype=np.uint64)
    for name, kw in (("nsl", dict(no_self_loops=True)), ("npe", dict(no_parallel_edges=True)),
                     ("both", dict(no_self_loops=True, no_parallel_edges=True))):
        f = pb.GenParams(n=n // 10, d=10, n0=12, seed_edges=seed, **kw)
        cf = f._device_params(dev)
        out = torch.empty(2 * (f.m - f.m0), dtype=torch.int64, device=dev)
        t = timeit(lambda: _lib.check(L.parba_generate(cf, f.m0, f.m, out.data_ptr(), prb.data_ptr(), st)), reps=6)
        res[f"flags_{name}_edges_per_s"] = (f.m - f.m0) / t
        del out
    print(json.dumps(res))


if __name__ == "__main__":
    main()
