"""Graph family and edge generation (reference: parba/generator.py).

Every edge of the derandomized Batagelj-Brandes array is a pure function of
its index: r := 2i+1; repeat r := h(r) until r is even (or falls into the
seed region r < 2*m0); the edge is (src(i), tgt(r)) (PAPER.md:100-105,
generator.py:139-181).  Here the chains run in the CUDA kernels of
``libparba_b200.so``; this module keeps the reference's names, validation,
argument meaning and return types so it is a drop-in for the plain
(uniform-degree) path.

Degree sequences (f4) run in the same tile kernels with owner lookups by
rank instead of the division by d (index built on the device by
``degreeseq``); the option flags no_self_loops / no_parallel_edges (f3) run in
the node-granular kernel (include/parba_b200.h, "Option flags").
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Literal, NamedTuple

import numpy as np

from . import _lib, degreeseq
from .errors import ParameterError
from .hashing import HashConfig, c_params

Resolution = Literal["rank", "bisect", "deferred"]

# degreeseq.py:27 -- largest supported edge count (positions stay < 2^59).
MAX_EDGES = 1 << 58

# Chunk of device output per launch when streaming a block back to the host
# (32 Mi edges = 512 MiB per buffer, two buffers in flight).
HOST_CHUNK_EDGES = 1 << 25

# Degree sequences: build the dense owner map (4 bytes per generated edge,
# one load per owner lookup instead of a rank entry + owners gather) when it
# fits in this many bytes and in a quarter of the free device memory.
DENSE_OWNER_MAX_BYTES = 1 << 34
DENSE_FORCE = False  # A/B (tools/degseq_lookup_ab.py): build the map without zero-degree nodes too


class Edge(NamedTuple):
    source: int
    target: int


class ChainResult(NamedTuple):
    """Terminal state of one chain (generator.py:38-47)."""

    half_pos: int | None
    seed_pos: int | None
    probes: int


@dataclass(frozen=True, eq=False)
class GenParams:
    """One member of the graph family (generator.py:50-133).

    Exactly one of d (uniform out-degree) and degrees must be given; the seed
    graph is a flat array of 2*m0 node IDs, all < n0.  Validation and derived
    quantities follow the reference.  Every family runs on the device:
    uniform degree and degree sequences (f4), with or without the option
    flags (f3), CRC or SIMPLE hash, salted or not.
    """

    n: int
    d: int | None = None
    degrees: np.ndarray | None = None
    n0: int = 0
    seed_edges: np.ndarray | None = None
    no_self_loops: bool = False
    no_parallel_edges: bool = False
    hash: HashConfig = field(default_factory=HashConfig)
    max_attempts: int | None = None

    def __post_init__(self) -> None:
        if (self.d is None) == (self.degrees is None):
            raise ParameterError("exactly one of d and degrees must be given")
        if self.n0 < 0 or self.n < self.n0:
            raise ParameterError(f"need 0 <= n0 <= n, got n0={self.n0}, n={self.n}")
        if self.d is not None and self.d < 1:
            raise ParameterError(f"uniform degree must be >= 1, got {self.d}")
        seed = np.array([] if self.seed_edges is None else self.seed_edges, dtype=np.uint64, copy=True)
        if seed.size % 2:
            raise ParameterError("seed_edges must hold two endpoints per edge")
        if seed.size and int(seed.max()) >= self.n0:
            raise ParameterError("seed graph references node IDs >= n0")
        object.__setattr__(self, "seed_edges", seed)
        if self.degrees is not None:
            degrees = np.asarray(self.degrees)
            if degrees.size != self.n - self.n0:
                raise ParameterError(
                    f"degree sequence length {degrees.size} != n - n0 = {self.n - self.n0}")
            degrees, m = degreeseq.validate_degrees(degrees, self.m0, self.n0)
            object.__setattr__(self, "degrees", np.array(degrees, dtype=np.uint64, copy=True))
            self.__dict__["_m"] = m
        if (self.no_self_loops or self.no_parallel_edges) and self.m0 < 1:
            raise ParameterError(
                "no_self_loops / no_parallel_edges require a seed graph (m0 >= 1): "
                "with an empty seed the first edge is the forced self-loop (0, 0)")
        if self.max_attempts is not None and self.max_attempts < 1:
            raise ParameterError("max_attempts must be >= 1")
        if self.m >= MAX_EDGES:
            raise ParameterError(f"total edge count {self.m} exceeds the supported maximum")

    @property
    def m0(self) -> int:
        return self.seed_edges.size // 2

    @property
    def m(self) -> int:
        if self.d is not None:
            return self.m0 + (self.n - self.n0) * self.d
        return self.__dict__["_m"]

    @property
    def prefix(self) -> "degreeseq.PrefixIndex":
        """Device prefix index of the degree sequence (generator.py:113-115)."""
        if self.d is not None:
            raise ParameterError("uniform-degree parameters have no prefix index")
        return self._index()[0]

    @property
    def rank_bits(self) -> "degreeseq.RankBits":
        if self.d is not None:
            raise ParameterError("uniform-degree parameters have no prefix index")
        return self._index()[1]

    def _index(self, device=None):
        """(prefix, rank bits, dense owner map or None) on `device` (cached)."""
        torch = _lib.torch_cuda()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        cache = self.__dict__.setdefault("_index_dev", {})
        key = (dev.type, dev.index)
        if key not in cache:
            pi = degreeseq.build_prefix(self.degrees, self.m0, self.n0, device=dev)
            rb = degreeseq.build_rank_bits(pi, device=dev)
            dense = None
            nbytes = 4 * (self.m - self.m0)
            # without zero-degree nodes a rank entry gives the owner directly
            # (one 16-byte load, with the skewed targets' low positions
            # L2-resident: 3.37e10 vs 2.94e10 edges/s through the dense map,
            # tools/degseq_lookup_ab.py); with zeros the rank path needs a
            # second (owners) gather and the dense map wins (2.96e10 vs 1.67e10)
            if ((rb.owners_dev is not None or DENSE_FORCE) and self.n < (1 << 32)
                    and 0 < nbytes <= DENSE_OWNER_MAX_BYTES):
                free, _ = torch.cuda.mem_get_info(dev)
                if nbytes <= free // 4:
                    dense = torch.empty(self.m - self.m0, dtype=torch.int32, device=dev)
                    with torch.cuda.device(dev):
                        _lib.check(_lib.load().parba_degseq_dense(pi.W_dev.data_ptr(), pi.n_nodes, self.m0,
                                                                  self.n0, dense.data_ptr(),
                                                                  _lib.stream_ptr(torch, dev)))
            cache[key] = (pi, rb, dense)
        return cache[key]

    def _host_W(self) -> np.ndarray:
        """Host prefix (node starts + m) for batch planning only."""
        W = self.__dict__.get("_W_host")
        if W is None:
            W = np.empty(self.degrees.size + 1, dtype=np.uint64)
            W[0] = self.m0
            np.cumsum(self.degrees, out=W[1:])
            W[1:] += np.uint64(self.m0)
            self.__dict__["_W_host"] = W
        return W

    def degree_of(self, v: int) -> int:
        if not self.n0 <= v < self.n:
            raise ParameterError(f"node {v} outside generated range [{self.n0}, {self.n})")
        if self.d is not None:
            return self.d
        return int(self.degrees[v - self.n0])

    def first_edge_of(self, v: int) -> int:
        if not self.n0 <= v < self.n:
            raise ParameterError(f"node {v} outside generated range [{self.n0}, {self.n})")
        if self.d is not None:
            return self.m0 + (v - self.n0) * self.d
        return int(self._host_W()[v - self.n0])

    @property
    def has_flags(self) -> bool:
        return self.no_self_loops or self.no_parallel_edges

    # -- device plumbing -----------------------------------------------------
    def _host_params(self):
        """(parba_params_t, keep-alive) with the seed graph in HOST memory, for
        the C ABI's host-buffer entry points (uniform degree only)."""
        seed = np.ascontiguousarray(self.seed_edges, dtype=np.uint64)
        cp = c_params(self.hash, self.n, self.d, self.n0, self.m0, seed.ctypes.data if seed.size else None)
        cp.flags = ((_lib.FLAG_NO_SELF_LOOPS if self.no_self_loops else 0)
                    | (_lib.FLAG_NO_PARALLEL_EDGES if self.no_parallel_edges else 0))
        cp.max_attempts = self.max_attempts or 0
        return cp, seed

    def _device_params(self, device) -> _lib.CParams:
        """parba_params_t with the seed graph (and a degree sequence's index)
        resident on `device` (cached)."""
        torch = _lib.torch_cuda()
        dev = torch.device(device)
        cache = self.__dict__.setdefault("_seed_dev", {})
        seed_ptr = None
        if self.m0:
            key = (dev.type, dev.index)
            if key not in cache:
                cache[key] = _lib.to_device_u64(torch, self.seed_edges, dev)
            seed_ptr = cache[key].data_ptr()
        if self.d is not None:
            cp = c_params(self.hash, self.n, self.d, self.n0, self.m0, seed_ptr)
        else:
            cp = c_params(self.hash, self.n, 1, self.n0, self.m0, seed_ptr)
            pi, rb, dense = self._index(dev)
            cp.d = 0
            cp.m = self.m
            cp.degree_prefix = pi.W_dev.data_ptr()
            cp.rank = rb.rank_dev.data_ptr() if rb.rank_dev is not None else None
            cp.owners = rb.owners_dev.data_ptr() if rb.owners_dev is not None else None
            cp.dense_owner = dense.data_ptr() if dense is not None else None
        cp.flags = ((_lib.FLAG_NO_SELF_LOOPS if self.no_self_loops else 0)
                    | (_lib.FLAG_NO_PARALLEL_EDGES if self.no_parallel_edges else 0))
        cp.max_attempts = self.max_attempts or 0
        return cp


def edge_count(p: GenParams) -> int:
    return p.m


def _check_resolution(resolution: str) -> None:
    if resolution not in degreeseq.RESOLVE:
        raise ParameterError(f"unknown resolution {resolution!r}")


def _cuts(p: GenParams, lo: int, hi: int, chunk: int) -> list[int]:
    """Chunk boundaries lo = c0 < c1 < ... = hi; node boundaries when an
    option flag makes generation node-granular (driver.py:131-158)."""
    if not p.has_flags:
        return list(range(lo, hi, chunk)) + [hi]
    cuts = [lo]
    if p.d is not None:
        step = max(p.d, (chunk // p.d) * p.d)
        a = lo
        while hi - a > step:
            a += step
            cuts.append(a)
    else:
        W = p._host_W()
        a = lo
        while hi - a > chunk:
            k = int(np.searchsorted(W, np.uint64(a + chunk), side="right")) - 1
            b = int(W[k])
            if b <= a:  # one node larger than a chunk
                k = int(np.searchsorted(W, np.uint64(a), side="right"))
                b = int(W[k]) if k < W.size else hi
            if b >= hi:
                break
            cuts.append(b)
            a = b
    return cuts + [hi]


def _device(device=None):
    torch = _lib.torch_cuda()
    if device is None:
        return torch, torch.device("cuda", torch.cuda.current_device())
    return torch, torch.device(device)


# ---------------------------------------------------------------------------
# Chains


def resolve_chain_block(r0, stop_below: int, cfg: HashConfig, device=None) -> tuple[np.ndarray, int]:
    """Kernel seam (_kernels.py:121-135): terminal r of every chain + total
    probes.  ``r0`` is not modified; a fresh uint64 array is returned."""
    r0 = np.ascontiguousarray(np.asarray(r0, dtype=np.uint64)).reshape(-1)
    if stop_below < 0 or stop_below > (1 << 64) - 1:
        raise ParameterError(f"stop_below out of range: {stop_below}")
    if r0.size == 0:
        return np.empty(0, dtype=np.uint64), 0
    if int(r0.min()) < 1:
        raise ParameterError(f"chain start must be >= 1, got {int(r0.min())}")
    torch, dev = _device(device)
    rd = _lib.to_device_u64(torch, r0, dev)
    out = torch.empty_like(rd)
    probes = torch.zeros(1, dtype=torch.int64, device=dev)
    L = _lib.load()
    with torch.cuda.device(dev):
        _lib.check(L.parba_resolve_chains(c_params(cfg), rd.data_ptr(), r0.size, stop_below,
                                          out.data_ptr(), probes.data_ptr(), _lib.stream_ptr(torch, dev)))
        return out.cpu().numpy().view(np.uint64), int(probes.item())


def resolve_chain(r0: int, stop_below: int, hash: HashConfig) -> ChainResult:
    """Scalar chain (generator.py:139-154) through the device kernel."""
    if r0 < 1:
        raise ParameterError(f"chain start must be >= 1, got {r0}")
    vals, probes = resolve_chain_block(np.array([r0], dtype=np.uint64), stop_below, hash)
    r = int(vals[0])
    if r < stop_below:
        return ChainResult(half_pos=None, seed_pos=r, probes=probes)
    return ChainResult(half_pos=r, seed_pos=None, probes=probes)


# ---------------------------------------------------------------------------
# Edges


def edges_at(ids, p: GenParams, device=None) -> tuple[np.ndarray, int]:
    """(k, 2) uint64 edges for an arbitrary list of edge IDs in [m0, m), plus
    total probes -- generate_edge vectorised (generator.py:172-181)."""
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64)).reshape(-1)
    if p.has_flags:
        raise ParameterError("option flags need whole-node processing; use generate_node_edges")
    if ids.size == 0:
        return np.empty((0, 2), dtype=np.uint64), 0
    lo_i, hi_i = int(ids.min()), int(ids.max())
    if lo_i < p.m0 or hi_i >= p.m:
        bad = lo_i if lo_i < p.m0 else hi_i
        raise ParameterError(f"edge index {bad} out of range [{p.m0}, {p.m})")
    torch, dev = _device(device)
    idd = _lib.to_device_u64(torch, ids, dev)
    out = torch.empty(2 * ids.size, dtype=torch.int64, device=dev)
    probes = torch.zeros(1, dtype=torch.int64, device=dev)
    L = _lib.load()
    with torch.cuda.device(dev):
        _lib.check(L.parba_edges_at(p._device_params(dev), idd.data_ptr(), ids.size, out.data_ptr(),
                                    probes.data_ptr(), _lib.stream_ptr(torch, dev)))
        return out.cpu().numpy().view(np.uint64).reshape(-1, 2), int(probes.item())


def generate_edge(i: int, p: GenParams) -> Edge:
    """Edge i in plain mode (generator.py:172-181)."""
    if p.no_self_loops or p.no_parallel_edges:
        raise ParameterError("option flags need whole-node processing; use generate_node_edges")
    if not p.m0 <= i < p.m:
        raise ParameterError(f"edge index {i} out of range [{p.m0}, {p.m})")
    e, _ = edges_at(np.array([i], dtype=np.uint64), p)
    return Edge(int(e[0, 0]), int(e[0, 1]))


def generate_node_edges(v: int, p: GenParams) -> list[Edge]:
    """All edges of node v in edge-index order, honouring the option flags
    (generator.py:220-228)."""
    if not p.n0 <= v < p.n:
        raise ParameterError(f"node {v} outside generated range [{p.n0}, {p.n})")
    first, dv = p.first_edge_of(v), p.degree_of(v)
    if dv == 0:
        return []
    if p.has_flags:
        e, _ = generate_block(first, first + dv, p)
    else:
        e, _ = edges_at(np.arange(first, first + dv, dtype=np.uint64), p)
    return [Edge(int(a), int(b)) for a, b in e]


def _check_block(lo: int, hi: int, p: GenParams) -> None:
    if not (p.m0 <= lo <= hi <= p.m):
        raise ParameterError(f"block [{lo}, {hi}) out of range [{p.m0}, {p.m}]")


def generate_block_device(lo: int, hi: int, p: GenParams, out=None, probes=None, device=None):
    """Store mode, device-resident: edges lo..hi-1 as an (hi-lo, 2) int64
    tensor holding the uint64 bits (IDs < 2^58), plus a device probe counter
    (incremented).  One launch of the tile kernel; asynchronous on the
    current stream."""
    _check_block(lo, hi, p)
    torch, dev = _device(device)
    if out is None:
        out = torch.empty((hi - lo, 2), dtype=torch.int64, device=dev)
    elif out.numel() < 2 * (hi - lo) or not out.is_contiguous() or out.device != dev:
        raise ParameterError("out must be a contiguous device tensor with 2*(hi-lo) int64 slots")
    if probes is None:
        probes = torch.zeros(1, dtype=torch.int64, device=dev)
    if hi > lo:
        L = _lib.load()
        with torch.cuda.device(dev):
            _lib.check(L.parba_generate(p._device_params(dev), lo, hi, out.data_ptr(), probes.data_ptr(),
                                        _lib.stream_ptr(torch, dev)))
    return out, probes


def generate_block(lo: int, hi: int, p: GenParams, resolution: Resolution = "rank",
                   device=None) -> tuple[np.ndarray, int]:
    """Edges lo..hi-1 as a fresh (hi-lo, 2) uint64 host array plus total
    probes (generator.py:258-325).

    Uniform degree: the C ABI's native host pipeline (``parba_generate_host``):
    the device generates only the u32 targets (CRC, no flags, n <= 2^32),
    they cross PCIe at 4 B per edge, and a team of host threads fills the
    (source, target) rows; other families stream 16-byte rows.  Degree
    sequences (their index lives on the device): device chunks streamed into
    pinned host memory while the next chunk is generated."""
    _check_block(lo, hi, p)
    _check_resolution(resolution)
    if lo == hi:
        return np.empty((0, 2), dtype=np.uint64), 0
    torch, dev = _device(device)
    total = hi - lo
    try:  # pinned (torch's caching host allocator: reused, already faulted in)
        out_host = torch.empty(2 * total, dtype=torch.int64, pin_memory=True)
    except RuntimeError:  # pinning refused (host limits): pageable array
        out_host = torch.empty(2 * total, dtype=torch.int64)
    L = _lib.load()
    if p.d is not None:
        import ctypes

        cp, _keep = p._host_params()
        probes = ctypes.c_uint64(0)
        idx = dev.index if dev.index is not None else torch.cuda.current_device()
        _lib.check(L.parba_generate_host(ctypes.byref(cp), lo, hi, out_host.data_ptr(), ctypes.byref(probes), idx))
        return out_host.numpy().view(np.uint64).reshape(-1, 2), int(probes.value)
    cuts = _cuts(p, lo, hi, min(total, HOST_CHUNK_EDGES))
    spans = list(zip(cuts, cuts[1:]))
    chunk = max(b - a for a, b in spans)
    with torch.cuda.device(dev):
        comp = torch.cuda.current_stream(dev)
        copy = torch.cuda.Stream(dev)
        bufs = [torch.empty(2 * chunk, dtype=torch.int64, device=dev) for _ in range(min(2, len(spans)))]
        probes = torch.zeros(1, dtype=torch.int64, device=dev)
        cp = p._device_params(dev)
        drained = [None, None]
        for k, (a, b) in enumerate(spans):
            buf = bufs[k % len(bufs)]
            if drained[k % 2] is not None:
                comp.wait_event(drained[k % 2])
            _lib.check(L.parba_generate(cp, a, b, buf.data_ptr(), probes.data_ptr(), comp.cuda_stream))
            made = torch.cuda.Event()
            made.record(comp)
            copy.wait_event(made)
            with torch.cuda.stream(copy):
                out_host[2 * (a - lo): 2 * (b - lo)].copy_(buf[: 2 * (b - a)], non_blocking=True)
                buf.record_stream(copy)
                ev = torch.cuda.Event()
                ev.record(copy)
                drained[k % 2] = ev
        copy.synchronize()
        nprobes = int(probes.item())
    return out_host.numpy().view(np.uint64).reshape(-1, 2), nprobes
