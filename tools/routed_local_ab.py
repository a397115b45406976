"""C4 full histogram on one GPU: the local n-word array (read-modify-write
flush) vs the owner-routed flush (red.add) into 1 / 8 slices on the same
GPU.  python tools/routed_local_ab.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1602_07106_b200 as pb

p = pb.GenParams(n=10**8, d=16)
dev = torch.device("cuda", 0)


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


counts = torch.zeros(p.n, dtype=torch.int32, device=dev)
prb = torch.zeros(1, dtype=torch.int64, device=dev)


def local():
    counts.zero_()
    pb.parallel.count_shard_device(p, p.n, 0, p.m, counts=counts, probes=prb, device=dev)


print(f"local array: {timeit(local):.3f} ms")
want = counts.clone()
for owners in (1, 8):
    S = pb.parallel.routed_slice_nodes(p.n, owners)
    whole = torch.zeros(S * owners, dtype=torch.int32, device=dev)
    ptrs = [whole[g * S:].data_ptr() for g in range(owners)]

    def routed():
        whole.zero_()
        pb.parallel.count_shard_routed(p, 0, p.m, ptrs, S, probes=prb, device=dev)

    t = timeit(routed)
    print(f"routed, {owners} slice(s): {t:.3f} ms, equal={bool((whole[:p.n] == want).all())}")
