"""Multi-GPU sharding: one process per GPU, ``torch.distributed`` (NCCL) for
the plumbing (reference counterpart: the fork workers and
``Consumer.merge`` of driver.py:210-270 / analytics.py:78-82).

Every edge is a pure function of its index, so rank g
of G takes the contiguous edge-ID shard

    [lo + floor(g*(hi-lo)/G), lo + floor((g+1)*(hi-lo)/G))

with no communication while generating.  Store mode needs no collective at
all; a degree count needs exactly one: the sum of the per-rank histograms
(NCCL reduce / all-reduce over NVLink).  Results are bit-identical for every
world size.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ParameterError


def world() -> tuple[int, int]:
    """(rank, world_size) of the default process group, (0, 1) without one."""
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return 0, 1
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_range(lo: int, hi: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous shard of [lo, hi) owned by `rank` (exact cover, no overlap)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ParameterError(f"bad rank {rank} of world {world_size}")
    if hi < lo:
        raise ParameterError(f"empty-or-negative range [{lo}, {hi})")
    n = hi - lo
    return lo + (rank * n) // world_size, lo + ((rank + 1) * n) // world_size


def node_floor(p, x: int) -> int:
    """Largest node boundary <= x (x in [m0, m]); m is a boundary."""
    if x >= p.m:
        return p.m
    if p.d is not None:
        return p.m0 + ((x - p.m0) // p.d) * p.d
    W = p._host_W()
    return int(W[int(np.searchsorted(W, np.uint64(x), side="right")) - 1])


def shard_range_for(p, lo: int, hi: int, rank: int, world_size: int) -> tuple[int, int]:
    """shard_range, with the cuts moved down to node boundaries when an
    option flag makes generation node-granular (lo, hi must be boundaries)."""
    a, b = shard_range(lo, hi, rank, world_size)
    if p.has_flags:
        a = lo if rank == 0 else max(lo, node_floor(p, a))
        b = hi if rank == world_size - 1 else max(lo, node_floor(p, b))
    return a, b


def reduce_counts(t, op: str = "allreduce", dst: int = 0, group=None):
    """Sum a per-rank count tensor over the group (NCCL on GPU tensors, gloo
    on CPU tensors).  ``op='reduce'`` leaves the sum on `dst` only."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return t
    if op == "allreduce":
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    elif op == "reduce":
        dist.reduce(t, dst=dst, op=dist.ReduceOp.SUM, group=group)
    else:
        raise ParameterError(f"unknown reduction {op!r}")
    return t


def count_shard_device(p, K: int, lo: int, hi: int, counts=None, probes=None, device=None):
    """Fused generate + count of edges [lo, hi) on one GPU.

    Returns (counts tensor, probes tensor).  K == n with 2m < 2^32 uses the
    uint32 full-histogram kernel; otherwise the uint64 window kernel."""
    from .generator import _device

    torch, dev = _device(device)
    L = _lib.load()
    full = (K == p.n and K > 0 and 2 * p.m < (1 << 32))
    if probes is None:
        probes = torch.zeros(1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        cp = p._device_params(dev)
        st = _lib.stream_ptr(torch, dev)
        if full:
            if counts is None:
                counts = torch.zeros(K, dtype=torch.int32, device=dev)
            _lib.check(L.parba_degree_full(cp, lo, hi, counts.data_ptr(), probes.data_ptr(), st))
        else:
            if counts is None:
                counts = torch.zeros(max(K, 1), dtype=torch.int64, device=dev)
            _lib.check(L.parba_degree_window(cp, lo, hi, K, counts.data_ptr() if K else None,
                                             probes.data_ptr(), st))
    return counts, probes


def widen_counts(torch, counts, K: int):
    """uint32 / int64 device counts -> int64 device tensor of length K."""
    if counts.dtype == torch.int32:
        return counts.to(torch.int64) & 0xFFFFFFFF
    return counts[:K]


def degree_counts_sharded(p, K: int, lo: int, hi: int, device=None):
    """This rank's shard of [lo, hi) counted on its GPU, summed over ranks.

    Returns (int64 numpy counts[K], total probes, per-rank [(rank, edges, probes)])."""
    from .generator import _device

    torch, dev = _device(device)
    rank, ws = world()
    a, b = shard_range_for(p, lo, hi, rank, ws)
    counts, probes = count_shard_device(p, K, a, b, device=dev)
    stats = torch.tensor([b - a, 0], dtype=torch.int64, device=dev)
    stats[1:2].copy_(probes)
    if ws > 1:
        # full histograms travel as 32-bit words (2m < 2^32, so the wrapped
        # int32 sum has the exact bits): half the bytes of an int64 reduce
        reduce_counts(counts)
        gathered = [torch.zeros_like(stats) for _ in range(ws)]
        import torch.distributed as dist

        dist.all_gather(gathered, stats)
        per = [(r, int(g[0].item()), int(g[1].item())) for r, g in enumerate(gathered)]
    else:
        per = [(0, b - a, int(probes.item()))]
    c64 = widen_counts(torch, counts, K)
    out = c64[:K].cpu().numpy() if K else np.zeros(0, dtype=np.int64)
    return out.astype(np.int64, copy=False), sum(pr for _, _, pr in per), per


_MULTI_MODES = {"store": _lib.MULTI_STORE, "window": _lib.MULTI_WINDOW, "full": _lib.MULTI_FULL,
                "discard": _lib.MULTI_DISCARD}


def multi_run(p, devices, mode: str = "window", K: int | None = None):
    """Whole graph [m0, m) on several GPUs from ONE process (C ABI
    ``parba_multi_run``: a host thread per device, counts summed on
    devices[0] over peer copies).  Returns (result, probes, device_seconds):
    result = (m - m0, 2) uint64 edges ('store'), int64 counts[K] ('window'),
    int64 counts[n] ('full') or None ('discard').  Uniform degree only."""
    import ctypes

    from .hashing import c_params

    if mode not in _MULTI_MODES:
        raise ParameterError(f"unknown mode {mode!r}")
    if p.d is None:
        raise ParameterError("multi_run takes uniform-degree families (degree sequences: one process per GPU)")
    devs = np.ascontiguousarray(np.asarray(list(devices), dtype=np.int32))
    if devs.size < 1:
        raise ParameterError("need at least one device")
    seed = np.ascontiguousarray(p.seed_edges, dtype=np.uint64)
    cp = c_params(p.hash, p.n, p.d, p.n0, p.m0, seed.ctypes.data if seed.size else None)
    cp.flags = ((_lib.FLAG_NO_SELF_LOOPS if p.no_self_loops else 0)
                | (_lib.FLAG_NO_PARALLEL_EDGES if p.no_parallel_edges else 0))
    cp.max_attempts = p.max_attempts or 0
    if mode == "window":
        K = p.n if K is None else K
        out = np.zeros(max(K, 1), dtype=np.int64)
    elif mode == "full":
        K = p.n
        out = np.zeros(max(K, 1), dtype=np.int64)
    elif mode == "store":
        K = 0
        out = np.empty((p.m - p.m0, 2), dtype=np.uint64)
    else:
        K, out = 0, None
    probes = ctypes.c_uint64(0)
    secs = ctypes.c_double(0.0)
    L = _lib.load()
    _lib.check(L.parba_multi_run(ctypes.byref(cp), int(devs.size), devs.ctypes.data, _MULTI_MODES[mode], K,
                                 out.ctypes.data if out is not None else None, ctypes.byref(probes),
                                 ctypes.byref(secs)))
    if mode in ("window", "full"):
        out = out[:K]
    return out, int(probes.value), float(secs.value)
