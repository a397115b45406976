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

import os

import numpy as np

from . import _lib
from .errors import GenerationError, ParameterError


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


def balanced_cuts(cuts, times, align: int = 256) -> list[int]:
    """Cut points of a contiguous partition re-balanced by measured cost.

    `cuts` (c_0 < ... <= c_N) is the partition a step ran with and `times`
    the N per-part device times.  The cost is taken as uniform inside each
    part (density t_k / (c_{k+1} - c_k)); the new cuts put 1/N of the total
    cost in every part (interior cuts rounded to multiples of `align`, the
    tile size).  The reference balances its workers dynamically (batches
    claimed from a shared cursor, driver.py:200-207); ranks of one
    collective need their ranges up front, so the balance is taken from a
    measured warm-up step instead.  Any cover of [c_0, c_N) gives the same
    counts."""
    n = len(times)
    if len(cuts) != n + 1 or n < 1:
        raise ParameterError("need N + 1 cuts for N times")
    lo, hi = int(cuts[0]), int(cuts[-1])
    if n == 1 or hi <= lo or min(times) <= 0:
        return [int(c) for c in cuts]
    total = float(sum(times))
    out = [lo]
    k, acc = 0, 0.0  # part k, cost before it
    for j in range(1, n):
        target = total * j / n
        while k < n - 1 and acc + times[k] < target:
            acc += times[k]
            k += 1
        a, b = int(cuts[k]), int(cuts[k + 1])
        x = a + (b - a) * min(1.0, max(0.0, (target - acc) / times[k]))
        x = int(round(x / align)) * align if align > 1 else int(round(x))
        out.append(min(hi, max(out[-1], x)))
    out.append(hi)
    return out


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


# --------------------------------------------------------------------------
# Owner-routed full histogram: the histogram reduce fused into the count
# kernels (include/parba_b200.h, parba_degree_full_routed).

MAX_OWNERS = 16


def routed_slice_nodes(n: int, owners: int) -> int:
    """Nodes per owner: ceil(n / owners) rounded up to a multiple of 2^16."""
    return ((n + owners - 1) // owners + 0xFFFF) & ~0xFFFF


def routed_ok(p, lo: int, hi: int, device=None) -> bool:
    """True when edges [lo, hi) can be counted straight into owner slices
    (plain uniform-degree family, n >= 2^25, a shard of >= 2^22 edges)."""
    from .generator import _device

    if p.d is None or p.has_flags or not (p.n < (1 << 32) and 2 * p.m < (1 << 32)):
        return False
    torch, dev = _device(device)
    with torch.cuda.device(dev):
        return bool(_lib.load().parba_degree_full_routed_ok(p._device_params(dev), lo, hi))


def count_shard_routed(p, lo: int, hi: int, slice_ptrs, slice_nodes: int, probes=None, device=None):
    """Generate edges [lo, hi) on this GPU and add the degree of every node v
    into owner v // slice_nodes's uint32 slice (``slice_ptrs[g]``: a device
    address valid on this GPU -- local, peer-mapped or IPC-mapped).  Returns
    the probes tensor.  The owners zero their slices before any caller starts
    and read them after every caller's stream has drained."""
    import ctypes

    from .generator import _device

    torch, dev = _device(device)
    if probes is None:
        probes = torch.zeros(1, dtype=torch.int64, device=dev)
    ptrs = (ctypes.c_void_p * len(slice_ptrs))(*[int(x) if x else None for x in slice_ptrs])
    with torch.cuda.device(dev):
        _lib.check(_lib.load().parba_degree_full_routed(p._device_params(dev), lo, hi, len(slice_ptrs), ptrs,
                                                        slice_nodes, probes.data_ptr(), _lib.stream_ptr(torch, dev)))
    return probes


class _RawU32:
    """A raw device allocation seen by torch (``torch.as_tensor``) without a copy."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<i4", "data": (ptr, False), "version": 2}


class RoutedCounts:
    """The full degree histogram reduce-scattered over the ranks of the
    default process group, one process per GPU: rank g owns the uint32
    counters of nodes [g*S, (g+1)*S) in plain device memory mapped into every
    other rank by CUDA IPC (NVLink peer memory), and every rank's count
    kernels add into the owners' slices as they go (no collective over an
    n-word array afterwards -- analytics.py:78-82's merge fused into the
    count).  ``run(lo, hi)``: zero -> barrier -> count -> drain + barrier;
    afterwards ``own`` (an int32 torch view of this rank's slice, bits of
    uint32 counts) is complete.  ``gather()`` returns the whole int64
    histogram on every rank (NCCL/gloo all-gather of the slices)."""

    def __init__(self, p, device=None, group=None):
        import ctypes

        import torch.distributed as dist

        from .generator import _device

        self.p, self.group = p, group
        self.torch, self.dev = _device(device)
        self.rank, self.ws = dist.get_rank(group), dist.get_world_size(group)
        if self.ws > MAX_OWNERS:
            raise ParameterError(f"routed counts take at most {MAX_OWNERS} owners")
        self.S = routed_slice_nodes(p.n, self.ws)
        L = _lib.load()
        self._ptr = ctypes.c_void_p()
        self._opened: list[int] = []
        self.ptrs: list[int] = []
        self.own = None
        self.error: str | None = None
        handle = ctypes.create_string_buffer(64)
        # every rank reaches every collective below even when a step failed
        # on it; `error` is then set on all ranks and the object is unusable
        try:
            with self.torch.cuda.device(self.dev):
                _lib.check(L.parba_ipc_alloc(self.S * 4, ctypes.byref(self._ptr), handle))
        except Exception as e:
            self.error = str(e)
        handles: list = [None] * self.ws
        mine = self.dev.index if self.dev.index is not None else self.torch.cuda.current_device()
        dist.all_gather_object(handles, None if self.error else (bytes(handle.raw), mine), group=group)
        if self.error is None and all(h is not None for h in handles):
            try:
                with self.torch.cuda.device(self.dev):
                    for g, (h, peer) in enumerate(handles):
                        if g == self.rank:
                            self.ptrs.append(self._ptr.value)
                            continue
                        # (ranks see the same device numbering under torchrun)
                        if peer != mine and not L.parba_peer_atomics_ok(mine, peer):
                            raise GenerationError(f"no native peer atomics between GPUs {mine} and {peer}")
                        q = ctypes.c_void_p()
                        _lib.check(L.parba_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(q)))
                        self._opened.append(q.value)
                        self.ptrs.append(q.value)
                self.own = self.torch.as_tensor(_RawU32(self._ptr.value, self.S), device=self.dev)
            except Exception as e:
                self.error = str(e)
        elif self.error is None:
            self.error = "a peer could not allocate its slice"
        errs: list = [None] * self.ws
        dist.all_gather_object(errs, self.error, group=group)
        bad = [f"rank {g}: {e}" for g, e in enumerate(errs) if e]
        if bad:
            self.error = "; ".join(bad)
            self.close()
        self.lo_node = self.rank * self.S
        self.count = max(0, min(self.S, p.n - self.lo_node))  # nodes of this rank's slice below n

    @classmethod
    def try_create(cls, p, device=None, group=None):
        """A RoutedCounts, or None on every rank when any rank could not set
        it up (no IPC / peer access between the GPUs): callers then reduce."""
        rc = cls(p, device=device, group=group)
        return None if rc.error else rc

    def run(self, lo: int, hi: int, probes=None):
        """Count edges [lo, hi) of this rank into the owners' slices.  Every
        rank of the group calls this (collective: two barriers)."""
        import torch.distributed as dist

        torch = self.torch
        self.own.zero_()
        torch.cuda.synchronize(self.dev)
        dist.barrier(group=self.group)  # every slice is zero before anyone adds
        probes = count_shard_routed(self.p, lo, hi, self.ptrs, self.S, probes=probes, device=self.dev)
        torch.cuda.synchronize(self.dev)
        dist.barrier(group=self.group)  # every rank's adds have landed
        return probes

    def gather(self):
        """int64 counts[n] on every rank."""
        import torch.distributed as dist

        own = self.own
        if dist.get_backend(self.group) == "gloo":  # gloo gathers host tensors only
            own = own.cpu()
        parts = [self.torch.empty_like(own) for _ in range(self.ws)]
        dist.all_gather(parts, own, group=self.group)
        c = self.torch.cat(parts)[: self.p.n].to(self.dev)
        return c.to(self.torch.int64) & 0xFFFFFFFF

    def close(self) -> None:
        import ctypes

        import torch.distributed as dist

        L = _lib.load()
        self.own = None
        with self.torch.cuda.device(self.dev):
            self.torch.cuda.synchronize(self.dev)
            for q in self._opened:
                L.parba_ipc_close(q)
            self._opened = []
            dist.barrier(group=self.group)  # no peer still maps this rank's slice
            if self._ptr:
                L.parba_ipc_free(self._ptr)
                self._ptr = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def widen_counts(torch, counts, K: int):
    """uint32 / int64 device counts -> int64 device tensor of length K."""
    if counts.dtype == torch.int32:
        return counts.to(torch.int64) & 0xFFFFFFFF
    return counts[:K]


def split_batches(n_batches: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous groups of batch indices, one per worker / rank:
    group w = batches [w*B//W, (w+1)*B//W) (empty when W > B).  The
    reference's workers claim batches from a shared cursor
    (driver.py:200-207); a contiguous static split keeps every worker's
    edges one range, so it runs as one fused launch."""
    return [(n_batches * w // parts, n_batches * (w + 1) // parts) for w in range(parts)]


def group_ranges(p, batches, groups) -> list[tuple[int, int]]:
    """Edge range [lo, hi) covered by each group of batches (empty: (m0, m0))."""
    return [(batches[a].lo, batches[b - 1].hi) if b > a else (p.m0, p.m0) for a, b in groups]


def worker_devices(workers: int, device=None) -> list[int]:
    """Device index of each worker: `device` for all of them when given,
    else the visible devices round-robin from the current one -- the
    reference's ``workers`` becomes a GPU count."""
    torch = _lib.torch_cuda()
    if device is not None:
        dev = torch.device(device)
        idx = dev.index if dev.index is not None else torch.cuda.current_device()
        return [idx] * workers
    n = torch.cuda.device_count()
    cur = torch.cuda.current_device()
    return [(cur + w) % n for w in range(workers)]


def _counts_kind(p, K: int) -> str:
    return "full" if (K == p.n and K > 0 and 2 * p.m < (1 << 32)) else "window"


def _run_one_device(p, mode: str, K: int, ranges, dev):
    """Every range on one device, back to back into one histogram (or one
    host array for 'store').  Returns (result, per-range probes)."""
    from .generator import _device, generate_block

    torch, dev = _device(dev)
    live = [(k, a, b) for k, (a, b) in enumerate(ranges) if b > a]
    probes = [0] * len(ranges)
    if mode == "store":
        parts = []
        for k, a, b in live:
            arr, probes[k] = generate_block(a, b, p, device=dev)
            parts.append(arr)
        if len(parts) == 1:
            return parts[0], probes
        return (np.concatenate(parts) if parts else np.empty((0, 2), dtype=np.uint64)), probes
    Kc = K if mode != "discard" else 0
    counts = None
    prb = torch.zeros(max(len(ranges), 1), dtype=torch.int64, device=dev)
    for k, a, b in live:
        counts, _ = count_shard_device(p, Kc, a, b, counts=counts, probes=prb[k:k + 1], device=dev)
    probes = [int(x) for x in prb.cpu().tolist()][: len(ranges)]
    if mode == "discard":
        return None, probes
    if counts is None or Kc == 0:
        return np.zeros(Kc, dtype=np.int64), probes
    c64 = widen_counts(torch, counts, Kc)
    return c64[:Kc].cpu().numpy().astype(np.int64, copy=False), probes


def run_shards(p, mode: str, K: int, ranges, devices):
    """Run shard k = edges ranges[k] on device devices[k] (single process).

    mode: 'window' (int64 counts[K]; K == n selects the u32 full-histogram
    kernels), 'discard', or 'store' ((sum, 2) uint64 rows of the ranges, in
    order -- the ranges must be contiguous).  Returns (result, per-shard
    probes).  One distinct device: the device path directly.  Several
    devices, uniform degree: the C ABI ``parba_multi_run_shards`` (a host
    thread per device, one NCCL reduce of the histograms).  Several devices
    with a degree sequence (its index lives on each device): a host thread per
    device, histograms summed on the host."""
    import ctypes

    if len(ranges) != len(devices):
        raise ParameterError("one device per shard")
    udev = list(dict.fromkeys(devices))
    if len(udev) == 1:
        return _run_one_device(p, mode, K, ranges, udev[0])
    if p.d is not None:
        cp, _keep = p._host_params()
        kind = {"store": _lib.MULTI_STORE, "discard": _lib.MULTI_DISCARD}.get(mode)
        if kind is None:
            kind = _lib.MULTI_FULL if _counts_kind(p, K) == "full" else _lib.MULTI_WINDOW
        lo_all = min(a for a, _ in ranges)
        hi_all = max(b for _, b in ranges)
        if kind == _lib.MULTI_STORE:
            out = np.empty((p.m - p.m0, 2), dtype=np.uint64)  # the C ABI writes edge i at row i - m0
        elif kind in (_lib.MULTI_WINDOW, _lib.MULTI_FULL):
            out = np.zeros(max(K, 1), dtype=np.int64)
        else:
            out = None
        devs = np.ascontiguousarray(devices, dtype=np.int32)
        los = np.ascontiguousarray([a for a, _ in ranges], dtype=np.uint64)
        his = np.ascontiguousarray([b for _, b in ranges], dtype=np.uint64)
        prs = np.zeros(len(ranges), dtype=np.uint64)
        secs = ctypes.c_double(0.0)
        L = _lib.load()
        _lib.check(L.parba_multi_run_shards(ctypes.byref(cp), len(ranges), devs.ctypes.data, los.ctypes.data,
                                            his.ctypes.data, kind, K if kind == _lib.MULTI_WINDOW else 0,
                                            out.ctypes.data if out is not None else None, prs.ctypes.data,
                                            ctypes.byref(secs)))
        if kind == _lib.MULTI_STORE:
            out = out[lo_all - p.m0: hi_all - p.m0]
        elif out is not None:
            out = out[:K]
        return out, [int(x) for x in prs]
    # degree sequence on several devices: a host thread per device, each
    # running its shards one by one (results kept per shard)
    import threading

    per: dict = {}
    errors: list = []

    def work(dv):
        try:
            for k, x in enumerate(devices):
                if x == dv:
                    res, pr = _run_one_device(p, mode, K, [ranges[k]], dv)
                    per[k] = (res, pr[0])
        except BaseException as e:  # re-raised below
            errors.append(e)

    ths = [threading.Thread(target=work, args=(dv,)) for dv in udev]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errors:
        raise errors[0]
    probes = [per[k][1] for k in range(len(ranges))]
    if mode == "store":
        return np.concatenate([per[k][0] for k in range(len(ranges))]), probes
    if mode == "discard":
        return None, probes
    return sum(per[k][0] for k in range(len(ranges))), probes


def multi_run(p, devices, mode: str = "window", K: int | None = None):
    """Whole graph [m0, m) on several GPUs from ONE process through the C ABI
    ``parba_multi_run`` (equal contiguous shards, a host thread per distinct
    device, one NCCL reduce).  Returns (result, probes, device_seconds):
    result = (m - m0, 2) uint64 edges ('store'), int64 counts[K] ('window'),
    int64 counts[n] ('full') or None ('discard').  Uniform degree only."""
    import ctypes

    modes = {"store": _lib.MULTI_STORE, "window": _lib.MULTI_WINDOW, "full": _lib.MULTI_FULL,
             "discard": _lib.MULTI_DISCARD}
    if mode not in modes:
        raise ParameterError(f"unknown mode {mode!r}")
    if p.d is None:
        raise ParameterError("multi_run takes uniform-degree families (degree sequences: one process per GPU)")
    devs = np.ascontiguousarray(np.asarray(list(devices), dtype=np.int32))
    if devs.size < 1:
        raise ParameterError("need at least one device")
    cp, _keep = p._host_params()
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
    _lib.check(L.parba_multi_run(ctypes.byref(cp), int(devs.size), devs.ctypes.data, modes[mode], K,
                                 out.ctypes.data if out is not None else None, ctypes.byref(probes),
                                 ctypes.byref(secs)))
    if mode in ("window", "full"):
        out = out[:K]
    return out, int(probes.value), float(secs.value)
