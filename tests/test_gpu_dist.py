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
