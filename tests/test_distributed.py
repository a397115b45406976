"""Multi-process host logic on CPU (gloo, world size 2): the edge-range
sharding and the histogram reduction the GPU path uses (parallel.py).  Each
rank counts its shard with the oracle (the GPU kernel's stand-in here: there is
no GPU in the CPU suite) and the ranks' histograms are summed with
parallel.reduce_counts -- the result must equal the single-process count, for
both the all-reduce and the reduce-to-root forms."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q) -> None:
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle as O
    from paper_1602_07106_b200 import parallel

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        assert parallel.world() == (rank, world)
        p = O.OParams(n=10**9, d=100)
        lo, hi, K = 5 * 10**9, 5 * 10**9 + 60_000, 10**5
        a, b = parallel.shard_range(lo, hi, rank, world)
        counts, probes = O.degree_block(p, a, b, K)
        t = torch.from_numpy(counts.copy())
        parallel.reduce_counts(t, op="allreduce")
        t2 = torch.from_numpy(counts.copy())
        parallel.reduce_counts(t2, op="reduce", dst=0)
        pr = torch.tensor([probes], dtype=torch.int64)
        dist.all_reduce(pr)
        # full histograms are reduced as 32-bit words: a per-rank count above
        # 2^31 wraps in int32 but the summed bits widen back to the exact total
        per_rank = 3_000_000_000 if rank == 0 else 1_000_000_000  # total 4e9 < 2^32
        w = torch.tensor([int(np.uint32(per_rank).view(np.int32)), 7], dtype=torch.int32)
        parallel.reduce_counts(w)
        wide = parallel.widen_counts(torch, w, 2)
        assert wide.tolist() == [4_000_000_000, 14]
        q.put((rank, (a, b), t.numpy().copy(), t2.numpy().copy(), int(pr.item())))
    finally:
        dist.destroy_process_group()


def test_sharded_window_counts_equal_single_process():
    import oracle as O

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = O.OParams(n=10**9, d=100)
    lo, hi, K = 5 * 10**9, 5 * 10**9 + 60_000, 10**5
    want, wp = O.degree_block(p, lo, hi, K)
    (r0, s0, all0, red0, pr0), (r1, s1, all1, red1, pr1) = res
    assert s0 == (lo, lo + 30_000) and s1 == (lo + 30_000, hi)  # exact cover
    assert np.array_equal(all0, want) and np.array_equal(all1, want)
    assert np.array_equal(red0, want)  # root holds the sum
    assert pr0 == pr1 == wp


def _worker_flags(rank: int, world: int, port: int, q) -> None:
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle as O
    import paper_1602_07106_b200 as pb
    from paper_1602_07106_b200 import parallel

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seed = (0, 1, 1, 2, 2, 3, 3, 0, 0, 2)
        deg = np.random.default_rng(2).integers(0, 6, size=3000).astype(np.uint64)
        deg[0] = 2
        p = pb.GenParams(n=3004, n0=4, degrees=deg, seed_edges=np.array(seed, dtype=np.uint64),
                         no_self_loops=True, no_parallel_edges=True)
        op = O.OParams(n=p.n, d=None, n0=4, seed_edges=seed, degrees=tuple(int(x) for x in deg),
                       no_self_loops=True, no_parallel_edges=True)
        a, b = parallel.shard_range_for(p, p.m0, p.m, rank, world)
        blk, probes = O.generate_block(op, a, b)  # node-aligned shard: no error
        counts = np.zeros(p.n, dtype=np.int64)
        O.count_block(counts, blk)
        t = torch.from_numpy(counts)
        parallel.reduce_counts(t, op="allreduce")
        pr = torch.tensor([probes], dtype=torch.int64)
        dist.all_reduce(pr)
        q.put((rank, (a, b), t.numpy().copy(), int(pr.item())))
    finally:
        dist.destroy_process_group()


def test_sharded_flag_counts_on_node_boundaries():
    """Option flags make shards node-granular (parallel.shard_range_for): the
    world-size-2 sum equals the single-process count of the whole graph."""
    import oracle as O

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_flags, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    seed = (0, 1, 1, 2, 2, 3, 3, 0, 0, 2)
    deg = np.random.default_rng(2).integers(0, 6, size=3000).astype(np.uint64)
    deg[0] = 2
    op = O.OParams(n=3004, d=None, n0=4, seed_edges=seed, degrees=tuple(int(x) for x in deg),
                   no_self_loops=True, no_parallel_edges=True)
    whole, wp = O.generate_block(op, op.m0, op.m)
    want = np.zeros(op.n, dtype=np.int64)
    O.count_block(want, whole)
    (r0, s0, c0, p0), (r1, s1, c1, p1) = res
    assert s0[0] == op.m0 and s0[1] == s1[0] and s1[1] == op.m
    assert np.array_equal(c0, want) and np.array_equal(c1, want) and p0 == p1 == wp
