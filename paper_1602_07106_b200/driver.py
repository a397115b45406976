"""Batch planning and execution (reference: parba/driver.py).

The reference cuts [m0, m) into batches claimed by forked CPU workers and
feeds each batch's (k, 2) array to a Python ``Consumer`` (driver.py:58-81,
161-270).  On the B200 path the consumers the hot path serves are fused into
device kernels instead:

  * ``DegreeCountConsumer``  -> the fused window / full-histogram kernels
  * ``CollectConsumer``      -> store mode (device array, streamed to host)
  * ``DiscardConsumer``      -> the streaming kernel with an empty window
  * ``io.EdgeFileWriter``    -> store mode streamed into the positional
                                binary file (cli.py:121-145)

Any other ``Consumer`` (a user plug-in, or a subclass of the built-in ones)
runs the reference's batch loop (driver.py:161-270): ``plan_batches`` cuts
[m0, m), ``workers`` host threads claim batches from a shared cursor, every
batch is generated on the GPU (``generate_block``) and handed to the
consumer's ``accept_block`` on the host, and the contexts are merged.  The
edges are still computed only by the CUDA kernels; the host runs the user's
consumer code.  Worker failures abort the run (GenerationError naming the
worker, or the original exception with one worker), as in the reference.

When ``torch.distributed`` is initialised the fused routes shard the edge
range over its ranks (one GPU each) and reduce histograms over NCCL --
results are identical for every workers / batch_size / world size, as in the
reference (driver.py:1-9).
"""

from __future__ import annotations

import enum
import os
import threading
import time
import traceback
from dataclasses import dataclass
from typing import Any, Sequence

import numpy as np

from .errors import GenerationError, ParameterError
from .generator import Edge, GenParams, Resolution

DEFAULT_BATCH_SIZE = 1 << 16  # driver.py:26


class Granularity(enum.Enum):
    EDGE = "edge"
    NODE = "node"


@dataclass(frozen=True)
class Batch:
    lo: int
    hi: int
    granularity: Granularity = Granularity.EDGE


@dataclass(frozen=True)
class WorkerStats:
    worker_id: int
    batches: int
    edges: int
    probes: int
    seconds: float


@dataclass(frozen=True)
class RunStats:
    edges_emitted: int
    hash_probes: int
    elapsed: float
    per_worker: tuple[WorkerStats, ...]


class Consumer:
    """Streaming edge consumer contract (driver.py:58-81)."""

    def new_context(self, worker_id: int) -> Any:
        return None

    def accept(self, ctx: Any, i: int, edge: Edge) -> None:
        raise NotImplementedError

    def accept_block(self, ctx: Any, lo: int, edges: np.ndarray) -> None:
        for k in range(edges.shape[0]):
            self.accept(ctx, lo + k, Edge(int(edges[k, 0]), int(edges[k, 1])))

    def finalize_context(self, ctx: Any) -> Any:
        return ctx

    def merge(self, contexts: Sequence[Any]) -> Any:
        raise NotImplementedError


class DiscardConsumer(Consumer):
    """Counts edges and drops them (driver.py:84-94)."""

    def new_context(self, worker_id: int) -> int:
        return 0

    def accept_block(self, ctx: int, lo: int, edges: np.ndarray) -> int:
        return ctx + edges.shape[0]

    def merge(self, contexts: Sequence[int]) -> int:
        return sum(contexts)


class CollectConsumer(Consumer):
    """Gathers all edges into one (m - m0, 2) array in edge-index order
    (driver.py:97-114)."""

    def new_context(self, worker_id: int) -> list:
        return []

    def accept_block(self, ctx: list, lo: int, edges: np.ndarray) -> list:
        ctx.append((lo, edges.copy()))
        return ctx

    def merge(self, contexts: Sequence[list]) -> np.ndarray:
        chunks = sorted((c for ctx in contexts for c in ctx), key=lambda c: c[0])
        if not chunks:
            return np.empty((0, 2), dtype=np.uint64)
        return np.concatenate([arr for _, arr in chunks])


def _round_down_to_node(p: GenParams, pos: int) -> int:
    if p.d is not None:
        return p.m0 + ((pos - p.m0) // p.d) * p.d
    W = p._host_W()  # cached prefix (the reference reuses p.prefix.W, driver.py:125-128)
    k = int(np.searchsorted(W, np.uint64(pos), side="right")) - 1
    return int(W[k])


def _next_node_boundary(p: GenParams, lo: int) -> int:
    if p.d is not None:
        return lo + p.d
    W = p._host_W()
    k = int(np.searchsorted(W, np.uint64(lo), side="right")) - 1
    return lo + int(p.degrees[k])


def plan_batches(p: GenParams, batch_size: int, granularity: Granularity | None = None) -> list[Batch]:
    """Cover [m0, m) exactly once with half-open batches (driver.py:131-158);
    node granularity rounds boundaries down to a node's first edge."""
    if batch_size < 1:
        raise ParameterError(f"batch_size must be >= 1, got {batch_size}")
    if granularity is None:
        node_gran = p.no_self_loops or p.no_parallel_edges
    else:
        node_gran = granularity is Granularity.NODE
    gran = Granularity.NODE if node_gran else Granularity.EDGE
    out = []
    lo = p.m0
    while lo < p.m:
        hi = min(lo + batch_size, p.m)
        if node_gran and hi < p.m:
            hi = _round_down_to_node(p, hi)
            if hi <= lo:
                hi = min(_next_node_boundary(p, lo), p.m)
        out.append(Batch(lo, hi, gran))
        lo = hi
    return out


def run(p: GenParams, consumer: Consumer, workers: int = 1, batch_size: int = DEFAULT_BATCH_SIZE,
        resolution: Resolution = "rank", device=None) -> tuple[Any, RunStats]:
    """Generate every edge of [m0, m) exactly once into a consumer.

    Returns (merged consumer result, RunStats) like driver.py:210-270.  The
    plan is the reference's (``plan_batches(p, batch_size)``); worker w takes
    the contiguous group of batches [w*B//W, (w+1)*B//W) and runs it as one
    fused launch on its GPU -- ``workers`` is a GPU count: the visible
    devices round-robin from the current one, or all on ``device`` when
    given (a device running several workers' groups runs them back to back).
    Several GPUs in one process go through the C ABI's multi-device driver
    (one NCCL reduce of the histograms).  Under an initialised
    ``torch.distributed`` world each rank is one worker instead (its group of
    batches on its GPU, histograms summed over NCCL).  ``RunStats.per_worker``
    has one entry per worker whose batch and edge counts add up to the plan."""
    from . import analytics, io, parallel
    from .generator import generate_block

    if workers < 1:
        raise ParameterError(f"workers must be >= 1, got {workers}")
    if batch_size < 1:
        raise ParameterError(f"batch_size must be >= 1, got {batch_size}")
    t0 = time.perf_counter()
    kind = type(consumer)
    if kind not in (analytics.DegreeCountConsumer, DiscardConsumer, io.EdgeFileWriter, CollectConsumer):
        return _run_generic(p, consumer, workers, batch_size, resolution, device, t0)
    batches = plan_batches(p, batch_size)
    rank, ws = parallel.world()
    if ws > 1:
        return _run_fused_ranks(p, consumer, batches, rank, ws, resolution, device, t0)
    groups = parallel.split_batches(len(batches), workers)
    ranges = parallel.group_ranges(p, batches, groups)
    devices = parallel.worker_devices(workers, device)
    if isinstance(consumer, analytics.DegreeCountConsumer):
        counts, probes = parallel.run_shards(p, "window", consumer.K, ranges, devices)
        merged = analytics.DegreeCounter(K=consumer.K, counts=counts)
    elif isinstance(consumer, DiscardConsumer):
        _, probes = parallel.run_shards(p, "discard", 0, ranges, devices)
        merged = p.m - p.m0
    elif isinstance(consumer, io.EdgeFileWriter):
        probes = _write_file_shards(p, consumer, ranges, devices)
        merged = 16 * (p.m - p.m0)
    elif workers == 1:  # CollectConsumer on one GPU: the host-array block path
        merged, pr = generate_block(p.m0, p.m, p, resolution=resolution, device=devices[0])
        probes = [pr]
    else:
        merged, probes = parallel.run_shards(p, "store", 0, ranges, devices)
    elapsed = time.perf_counter() - t0
    per_worker = tuple(WorkerStats(w, b - a, r1 - r0, pr, elapsed)
                       for w, ((a, b), (r0, r1), pr) in enumerate(zip(groups, ranges, probes)))
    return merged, RunStats(edges_emitted=sum(w.edges for w in per_worker),
                            hash_probes=sum(w.probes for w in per_worker),
                            elapsed=elapsed, per_worker=per_worker)


def _write_file_shards(p: GenParams, consumer, ranges, devices) -> list[int]:
    """EdgeFileWriter: each worker's range written from its device (a host
    thread per distinct device; positional writes, so any order)."""
    probes = [0] * len(ranges)
    errors: list = []

    def work(dv):
        try:
            for k, (a, b) in enumerate(ranges):
                if devices[k] == dv and b > a:
                    probes[k] = consumer.write_range(p, a, b, device=dv)[1]
        except BaseException as e:  # re-raised below
            errors.append(e)

    udev = list(dict.fromkeys(devices))
    if len(udev) == 1:
        work(udev[0])
    else:
        ths = [threading.Thread(target=work, args=(dv,)) for dv in udev]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    if errors:
        raise errors[0]
    return probes


def _run_fused_ranks(p: GenParams, consumer, batches, rank: int, ws: int, resolution, device, t0):
    """One worker per torch.distributed rank: this rank's group of batches on
    its GPU; histograms summed over NCCL, stats all-gathered."""
    import torch.distributed as dist

    from . import analytics, io, parallel
    from .generator import _device, generate_block

    torch, dev = _device(device)
    groups = parallel.split_batches(len(batches), ws)
    a, b = parallel.group_ranges(p, batches, [groups[rank]])[0]
    counts = None
    if isinstance(consumer, (analytics.DegreeCountConsumer, DiscardConsumer)):
        K = consumer.K if isinstance(consumer, analytics.DegreeCountConsumer) else 0
        prb = torch.zeros(1, dtype=torch.int64, device=dev)
        full = bool(K) and parallel._counts_kind(p, K) == "full"
        routed = None
        if full and os.environ.get("PARBA_ROUTED", "1") != "0":
            # full histogram: the reduce fused into the count kernels (every
            # rank adds into the owners' slices over peer memory) when the
            # path applies to every rank's shard and the GPUs can map each other
            ok = torch.tensor([1 if (b == a or parallel.routed_ok(p, a, b, dev)) else 0], dtype=torch.int32,
                              device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()):
                routed = parallel.RoutedCounts.try_create(p, device=dev)
        if routed is not None:
            with routed:
                routed.run(a, b, probes=prb)
                counts = routed.gather()  # int64, the whole histogram on every rank
            if int(counts.sum().item()) != 2 * (p.m - p.m0):  # every endpoint landed in a slice
                raise GenerationError("owner-routed degree counts lost endpoints (peer atomics); "
                                      "set PARBA_ROUTED=0 to count locally and reduce")
        else:
            if K:
                counts = torch.zeros(K, dtype=torch.int32 if full else torch.int64, device=dev)
            if b > a:
                counts, _ = parallel.count_shard_device(p, K, a, b, counts=counts, probes=prb, device=dev)
            if K:
                # full histograms travel as 32-bit words (2m < 2^32, so the wrapped
                # int32 sum has the exact bits): half the bytes of an int64 reduce
                parallel.reduce_counts(counts)
        probes = int(prb.item())
        if isinstance(consumer, analytics.DegreeCountConsumer):
            c = (parallel.widen_counts(torch, counts, K)[:K].cpu().numpy() if K
                 else np.zeros(0, dtype=np.int64))
            merged = analytics.DegreeCounter(K=K, counts=c)
        else:
            merged = p.m - p.m0
    elif isinstance(consumer, io.EdgeFileWriter):
        dist.barrier()  # every rank has opened (and rank 0 sized) the file
        probes = consumer.write_range(p, a, b, device=dev)[1] if b > a else 0
        dist.barrier()  # the file is complete on return
        merged = 16 * (p.m - p.m0)
    else:  # CollectConsumer: the merged array is the whole graph on every rank;
        # this rank's stats are its own group's share of the plan
        parts, probes = [], 0
        for x, y in ((p.m0, a), (a, b), (b, p.m)):
            if y > x:
                arr, pr = generate_block(x, y, p, resolution=resolution, device=dev)
                parts.append(arr)
                probes += pr if (x, y) == (a, b) else 0
        merged = np.concatenate(parts) if parts else np.empty((0, 2), dtype=np.uint64)
    elapsed = time.perf_counter() - t0
    t = torch.tensor([groups[rank][1] - groups[rank][0], b - a, probes], dtype=torch.int64, device=dev)
    gathered = [torch.zeros_like(t) for _ in range(ws)]
    dist.all_gather(gathered, t)
    per_worker = tuple(WorkerStats(r, int(g[0].item()), int(g[1].item()), int(g[2].item()), elapsed)
                       for r, g in enumerate(gathered))
    return merged, RunStats(edges_emitted=sum(w.edges for w in per_worker),
                            hash_probes=sum(w.probes for w in per_worker),
                            elapsed=elapsed, per_worker=per_worker)


def _run_generic(p: GenParams, consumer: Consumer, workers: int, batch_size: int, resolution: Resolution,
                 device, t0: float) -> tuple[Any, RunStats]:
    """The reference's batch loop (driver.py:161-270) with host threads as
    workers and the GPU generating every batch."""
    from .generator import generate_block

    batches = plan_batches(p, batch_size)
    lock = threading.Lock()
    cursor = [0]
    abort = threading.Event()

    def claim() -> int:
        with lock:
            k = cursor[0]
            cursor[0] = k + 1
            return k

    def work(worker_id: int):
        start = time.perf_counter()
        ctx = consumer.new_context(worker_id)
        nb = edges = probes = 0
        while not abort.is_set():
            k = claim()
            if k >= len(batches):
                break
            b = batches[k]
            arr, pr = generate_block(b.lo, b.hi, p, resolution=resolution, device=device)
            ret = consumer.accept_block(ctx, b.lo, arr)
            if ret is not None:
                ctx = ret
            nb += 1
            edges += b.hi - b.lo
            probes += pr
        stats = WorkerStats(worker_id, nb, edges, probes, time.perf_counter() - start)
        return consumer.finalize_context(ctx), stats

    if workers == 1:
        result, st = work(0)
        results, per_worker = [result], [st]
    else:
        out: list = [None] * workers
        errors: list = []

        def main(w: int) -> None:
            try:
                out[w] = work(w)
            except BaseException:
                abort.set()
                errors.append((w, traceback.format_exc()))

        threads = [threading.Thread(target=main, args=(w,), daemon=True) for w in range(workers)]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        if errors:
            w, tb = sorted(errors)[0]
            raise GenerationError(f"worker {w} failed:\n{tb}")
        results = [o[0] for o in out]
        per_worker = [o[1] for o in out]
    merged = consumer.merge(results)
    return merged, RunStats(edges_emitted=sum(w.edges for w in per_worker),
                            hash_probes=sum(w.probes for w in per_worker),
                            elapsed=time.perf_counter() - t0, per_worker=tuple(per_worker))
