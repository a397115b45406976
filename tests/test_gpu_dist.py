"""``run`` / ``degree_counts`` under an initialised torch.distributed world
(driver._run_fused_ranks: each rank one worker, its group of batches on its
GPU, histograms summed by the collective, RunStats all-gathered).

Control-flow check on ONE GPU: two gloo ranks share cuda:0 (gloo reduces on
the host, so no kernel waits on another rank's kernel).  Results must equal
the single-process run, and the stats must cover the reference plan."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank: int, world: int, port: int, path: str, q) -> None:
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import paper_1602_07106_b200 as pb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tri = np.array([0, 1, 1, 2, 2, 0], dtype=np.uint64)
        p = pb.GenParams(n=40_000, d=5, n0=3, seed_edges=tri)
        full, fst = pb.degree_counts(p, batch_size=5000)
        win, _ = pb.degree_counts(p, K=777, batch_size=5000)
        n_disc, dst = pb.run(p, pb.DiscardConsumer(), batch_size=5000)
        arr, cst = pb.run(p, pb.CollectConsumer(), batch_size=5000)
        with pb.EdgeFileWriter(path, p.m0, p.m - p.m0, create=(rank == 0)) as w:
            nbytes, _ = pb.run(p, w, batch_size=5000)
        q.put((rank, full.counts, win.counts, n_disc, arr, nbytes,
               [(s.worker_id, s.batches, s.edges, s.probes) for s in fst.per_worker], fst.hash_probes,
               [(s.worker_id, s.batches, s.edges) for s in cst.per_worker]))
    finally:
        dist.destroy_process_group()


def test_run_under_torch_distributed(tmp_path):
    import torch.multiprocessing as mp

    import paper_1602_07106_b200 as pb

    path = str(tmp_path / "edges.bin")
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, world, port, path, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    tri = np.array([0, 1, 1, 2, 2, 0], dtype=np.uint64)
    p = pb.GenParams(n=40_000, d=5, n0=3, seed_edges=tri)
    full, fst = pb.degree_counts(p, batch_size=5000)
    win, _ = pb.degree_counts(p, K=777, batch_size=5000)
    want, _ = pb.generate_block(p.m0, p.m, p)
    plan = pb.plan_batches(p, 5000)
    for r in res:
        _, c, w, nd, arr, nbytes, per, probes, cper = r
        assert np.array_equal(c, full.counts) and np.array_equal(w, win.counts)
        assert nd == p.m - p.m0 and np.array_equal(arr, want) and nbytes == 16 * (p.m - p.m0)
        assert [x[0] for x in per] == [0, 1] and sum(x[1] for x in per) == len(plan)
        assert sum(x[2] for x in per) == p.m - p.m0 and probes == fst.hash_probes
        assert sum(x[1] for x in cper) == len(plan)
    assert np.array_equal(np.fromfile(path, dtype="<u8").reshape(-1, 2), want)


def _rank_routed(rank: int, world: int, port: int, q) -> None:
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["PARBA_FULL_MODE"] = "partition"  # the partitioned pass at test size
    import torch
    import torch.distributed as dist

    import paper_1602_07106_b200 as pb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tri = np.array([0, 1, 1, 2, 2, 0], dtype=np.uint64)
        p = pb.GenParams(n=300_000, d=5, n0=3, seed_edges=tri)
        a, b = pb.parallel.shard_range(p.m0, p.m, rank, world)
        rc = pb.parallel.RoutedCounts.try_create(p, device="cuda:0")
        if rc is None:
            q.put((rank, None, None, None, None))
            return
        with rc:
            prb = rc.run(a, b)
            own = (rc.own[: rc.count].to(torch.int64) & 0xFFFFFFFF).cpu().numpy()
            lo_node = rc.lo_node
            whole = rc.gather().cpu().numpy()
            prb2 = rc.run(a, b)  # a second step into re-zeroed slices
            again = rc.gather().cpu().numpy()
        assert np.array_equal(whole, again) and int(prb.item()) == int(prb2.item()) > 0
        full, st = pb.degree_counts(p)  # driver path: routed, then gathered
        q.put((rank, lo_node, own, whole, full.counts))
    finally:
        dist.destroy_process_group()


def test_routed_counts_two_ranks_ipc():
    """RoutedCounts over two processes sharing cuda:0: each rank owns a slice
    mapped into the other by CUDA IPC and both count into both slices.
    (Host barriers only: no kernel waits on another rank's kernel.)"""
    import torch.multiprocessing as mp

    import paper_1602_07106_b200 as pb

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_routed, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    if res[0][1] is None:
        pytest.skip("CUDA IPC between two processes is not available on this box")
    tri = np.array([0, 1, 1, 2, 2, 0], dtype=np.uint64)
    p = pb.GenParams(n=300_000, d=5, n0=3, seed_edges=tri)
    want, _ = pb.degree_counts(p)
    gen = want.counts.copy()  # the generated edges alone: degree_counts adds the seed graph's
    np.subtract.at(gen, tri.astype(np.int64), 1)
    for rank, lo_node, own, whole, full in res:
        assert np.array_equal(whole, gen) and np.array_equal(full, want.counts)
        assert np.array_equal(own, gen[lo_node: lo_node + len(own)])
    assert sum(len(r[2]) for r in res) == p.n
