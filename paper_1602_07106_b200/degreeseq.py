"""Degree-sequence index on the device (reference: parba/degreeseq.py).

With individual degrees the source of edge ``e`` is the node ``v`` with
``W[v] <= e < W[v] + d_v`` (W = prefix sums of the degrees).  The reference
offers three interchangeable lookups -- a rank bit vector, binary search over
W, and a deferred sort-and-merge -- and so does this module, all computed by
the CUDA library (``parba_degseq_prefix`` / ``parba_degseq_rank`` /
``parba_node_of_edges``, include/parba_b200.h):

  * W is an exclusive scan on the device (CUB) -- degreeseq.py:87-115;
  * the rank directory keeps one 16-byte entry per 64 positions (start bits
    plus the count of ones before the word), so a lookup is one 16-byte load
    and a popcount instead of the reference's word + superblock + offset
    reads (degreeseq.py:118-162);
  * bisect and deferred run as device kernels (the deferred path sorts with a
    CUB radix sort and merges runs against W) -- degreeseq.py:188-216.

Input validation (dtype, sign, overflow, the 2^58 cap) is host logic and
follows build_prefix exactly.  ``PrefixIndex.W`` / ``RankBits.words`` are
host copies of the device arrays for inspection; the generator kernels read
the device copies.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ParameterError

# Node degrees for nodes n0..n-1, one entry per node, zeros permitted.
DegreeSequence = np.ndarray

# degreeseq.py:27 -- half-open cap keeping 2*m and 16*(m - m0) inside int64.
MAX_EDGES = 1 << 58

RESOLVE = {"rank": 0, "bisect": 1, "deferred": 2}


def validate_degrees(degrees, m0: int, n0: int) -> tuple[np.ndarray, int]:
    """build_prefix's checks (degreeseq.py:87-109): returns (uint64 degrees, m)."""
    degrees = np.asarray(degrees)
    if degrees.ndim != 1:
        raise ParameterError("degree sequence must be one-dimensional")
    if degrees.size and degrees.dtype.kind not in "ui":
        raise ParameterError("degrees must be integers")
    if degrees.dtype.kind == "i" and degrees.size and int(degrees.min()) < 0:
        raise ParameterError("degrees must be non-negative")
    if m0 < 0 or n0 < 0:
        raise ParameterError("m0 and n0 must be non-negative")
    degrees = degrees.astype(np.uint64, copy=False)
    if degrees.size:
        csum = np.cumsum(degrees)
        # each degree fits in 64 bits, so a wraparound shows as a decreasing step
        if np.any(csum[1:] < csum[:-1]):
            raise ParameterError("degree sequence overflows the edge index space")
        total = int(csum[-1])
    else:
        total = 0
    m = m0 + total
    if m >= MAX_EDGES:
        raise ParameterError(f"total edge count {m} exceeds the supported maximum")
    return degrees, m


def _device(device=None):
    torch = _lib.torch_cuda()
    if device is None:
        return torch, torch.device("cuda", torch.cuda.current_device())
    return torch, torch.device(device)


@dataclass(frozen=True, eq=False)
class PrefixIndex:
    """Prefix sums of a degree sequence (degreeseq.py:47-66).

    ``W[v - n0]`` is node v's first edge; ``m`` counts the seed's m0 edges too.
    ``W_dev`` is the device array (n_nodes + 1 entries, the last one m)."""

    W: np.ndarray
    degrees: np.ndarray
    m: int
    m0: int
    n0: int
    W_dev: object = field(default=None, repr=False)

    @property
    def n_nodes(self) -> int:
        return len(self.W)


@dataclass(frozen=True, eq=False)
class RankBits:
    """Rank directory of a PrefixIndex (degreeseq.py:69-84), on the device.

    ``rank_dev``: (nwords, 2) int64 tensor {start bits, ones before the word};
    ``owners_dev``: rank -> node map, None when every node owns an edge."""

    nbits: int
    n_ones: int
    n0: int
    m0: int
    rank_dev: object = field(repr=False)
    owners_dev: object = field(default=None, repr=False)
    prefix: PrefixIndex | None = field(default=None, repr=False)

    @property
    def words(self) -> np.ndarray:
        """Bit words (bit j of word w = a node starts at 64w + j)."""
        if self.rank_dev is None:
            return np.zeros(0, dtype=np.uint64)
        return self.rank_dev[:, 0].cpu().numpy().view(np.uint64)

    @property
    def owners(self) -> np.ndarray | None:
        if self.owners_dev is None:
            return None
        return self.owners_dev.cpu().numpy().view(np.uint64)


def build_prefix(degrees: DegreeSequence, m0: int, n0: int, device=None) -> PrefixIndex:
    """W on the device by an exclusive scan (degreeseq.py:87-115)."""
    degrees, m = validate_degrees(degrees, m0, n0)
    torch, dev = _device(device)
    L = _lib.load()
    with torch.cuda.device(dev):
        W = torch.empty(degrees.size + 1, dtype=torch.int64, device=dev)
        deg_d = _lib.to_device_u64(torch, degrees, dev) if degrees.size else None
        _lib.check(L.parba_degseq_prefix(deg_d.data_ptr() if deg_d is not None else None, degrees.size, m0,
                                         W.data_ptr(), _lib.stream_ptr(torch, dev)))
        W_host = W.cpu().numpy().view(np.uint64)
    if int(W_host[-1]) != m:  # the device scan and the host total must agree
        raise ParameterError(f"degree prefix total {int(W_host[-1])} != {m}")
    return PrefixIndex(W=W_host[:-1].copy(), degrees=degrees, m=m, m0=m0, n0=n0, W_dev=W)


def build_rank_bits(pi: PrefixIndex, device=None) -> RankBits:
    """Rank directory over positions [0, m) (degreeseq.py:118-151)."""
    torch, dev = _device(device if device is not None else (pi.W_dev.device if pi.W_dev is not None else None))
    L = _lib.load()
    nwords = (pi.m + 63) // 64
    zero_deg = bool(pi.degrees.size) and int(pi.degrees.min()) == 0
    with torch.cuda.device(dev):
        rank = torch.empty((max(nwords, 1), 2), dtype=torch.int64, device=dev)
        owners = torch.empty(max(pi.n_nodes, 1), dtype=torch.int64, device=dev) if zero_deg else None
        n_ones = _lib.ctypes.c_uint64(0)
        _lib.check(L.parba_degseq_rank(pi.W_dev.data_ptr(), pi.n_nodes, pi.m, pi.n0, rank.data_ptr(),
                                       owners.data_ptr() if owners is not None else None,
                                       _lib.ctypes.byref(n_ones), _lib.stream_ptr(torch, dev)))
    n1 = int(n_ones.value)
    if owners is not None:
        owners = owners[:n1]
    return RankBits(nbits=pi.m, n_ones=n1, n0=pi.n0, m0=pi.m0, rank_dev=rank[:nwords] if nwords else None,
                    owners_dev=owners, prefix=pi)


def _ids(es) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(es, dtype=np.uint64)).reshape(-1)


def rank1_many(rb: RankBits, es) -> np.ndarray:
    """Ones at positions 0..e inclusive, per e (degreeseq.py:154-162)."""
    es = _ids(es)
    if es.size == 0:
        return np.zeros(0, dtype=np.uint64)
    if int(es.max()) >= rb.nbits:
        raise ParameterError(f"rank position {int(es.max())} out of range [0, {rb.nbits})")
    torch = _lib.torch_cuda()
    dev = rb.rank_dev.device
    L = _lib.load()
    with torch.cuda.device(dev):
        ed = _lib.to_device_u64(torch, es, dev)
        out = torch.empty_like(ed)
        _lib.check(L.parba_rank1(rb.rank_dev.data_ptr(), ed.data_ptr(), es.size, out.data_ptr(),
                                 _lib.stream_ptr(torch, dev)))
        return out.cpu().numpy().view(np.uint64)


def rank1(rb: RankBits, e: int) -> int:
    if not 0 <= e < rb.nbits:
        raise ParameterError(f"rank position {e} out of range [0, {rb.nbits})")
    return int(rank1_many(rb, np.array([e], dtype=np.uint64))[0])


def _lookup(es, pi: PrefixIndex, rb: RankBits | None, method: str) -> np.ndarray:
    es = _ids(es)
    if es.size == 0:
        return np.zeros(0, dtype=np.uint64)
    lo_e, hi_e = int(es.min()), int(es.max())
    if lo_e < pi.m0 or hi_e >= pi.m:
        bad = lo_e if lo_e < pi.m0 else hi_e
        raise ParameterError(f"edge index {bad} out of generated range [{pi.m0}, {pi.m})")
    if rb is None:
        rb = pi.__dict__.get("_rank_bits")
        if rb is None:
            rb = pi.__dict__["_rank_bits"] = build_rank_bits(pi)
    torch = _lib.torch_cuda()
    dev = pi.W_dev.device
    L = _lib.load()
    cp = index_params(pi, rb)
    with torch.cuda.device(dev):
        ed = _lib.to_device_u64(torch, es, dev)
        out = torch.empty_like(ed)
        _lib.check(L.parba_node_of_edges(cp, ed.data_ptr(), es.size, out.data_ptr(), RESOLVE[method],
                                         _lib.stream_ptr(torch, dev)))
        return out.cpu().numpy().view(np.uint64)


def index_params(pi: PrefixIndex, rb: RankBits) -> "_lib.CParams":
    """A parba_params_t carrying just the index (lookups need no hash)."""
    p = _lib.CParams()
    p.n = pi.n0 + pi.n_nodes
    p.d = 0
    p.n0 = pi.n0
    p.m0 = pi.m0
    p.m = pi.m
    p.degree_prefix = pi.W_dev.data_ptr()
    p.rank = rb.rank_dev.data_ptr() if rb.rank_dev is not None else None
    p.owners = rb.owners_dev.data_ptr() if rb.owners_dev is not None else None
    if p.m0:  # validation needs a seed pointer when m0 > 0; lookups never read it
        p.seed_edges = pi.W_dev.data_ptr()
    return p


def node_of_edge_many(es, rb: RankBits) -> np.ndarray:
    """Owning nodes by rank (degreeseq.py:181-185)."""
    return _lookup(es, rb.prefix, rb, "rank")


def node_of_edge(e: int, rb: RankBits) -> int:
    if not rb.m0 <= e < rb.nbits:
        raise ParameterError(f"edge index {e} out of generated range [{rb.m0}, {rb.nbits})")
    return int(node_of_edge_many(np.array([e], dtype=np.uint64), rb)[0])


def node_of_edge_bisect_many(es, pi: PrefixIndex) -> np.ndarray:
    """Owning nodes by binary search over W (degreeseq.py:199-201)."""
    return _lookup(es, pi, None, "bisect")


def node_of_edge_bisect(e: int, pi: PrefixIndex) -> int:
    if not pi.m0 <= e < pi.m:
        raise ParameterError(f"edge index {e} out of generated range [{pi.m0}, {pi.m})")
    return int(node_of_edge_bisect_many(np.array([e], dtype=np.uint64), pi)[0])


def owners_of_edges_deferred(es, pi: PrefixIndex) -> np.ndarray:
    """Owning nodes via device radix sort + merge against W + scatter back
    (degreeseq.py:204-216)."""
    return _lookup(es, pi, None, "deferred")


def resolve_targets_deferred(pairs: list[tuple[int, int]], pi: PrefixIndex) -> list[tuple[int, int]]:
    """(edge index i, even terminal half-position r) -> (source, target)
    (degreeseq.py:219-240)."""
    if not pairs:
        return []
    for i, r in pairs:
        if r & 1:
            raise ParameterError(f"terminal half-position {r} for edge {i} is odd")
        if r >> 1 >= pi.m:
            raise ParameterError(f"terminal half-position {r} out of range")
    idx = np.array([i for i, _ in pairs], dtype=np.uint64)
    half = np.array([r >> 1 for _, r in pairs], dtype=np.uint64)
    sources = owners_of_edges_deferred(idx, pi)
    # a position inside the seed region merges to the first block, as in the
    # reference's linear merge (_kernels.py:101-118); callers map seed
    # targets themselves
    gen = half >= np.uint64(pi.m0)
    targets = np.full(half.size, pi.n0, dtype=np.uint64)
    if gen.any():
        targets[gen] = owners_of_edges_deferred(half[gen], pi)
    return [(int(u), int(v)) for u, v in zip(sources, targets)]


def first_half_pos(v: int, pi: PrefixIndex) -> int:
    """Chain start 2*W[v] for self-loop avoidance (degreeseq.py:243-250)."""
    k = v - pi.n0
    if not 0 <= k < pi.n_nodes:
        raise ParameterError(f"node {v} outside generated range")
    if int(pi.degrees[k]) == 0:
        raise ParameterError(f"node {v} has degree zero and owns no edges")
    return 2 * int(pi.W[k])


def read_degree_file(path: str) -> DegreeSequence:
    """One decimal degree per line; line v gives node n0+v's degree
    (degreeseq.py:253-264)."""
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().split("\n")
    while lines and lines[-1].strip() == "":
        lines.pop()
    degrees = []
    for line_no, raw in enumerate(lines, start=1):
        s = raw.strip()
        if not (s.isascii() and s.isdigit()):
            raise ParameterError(f"{path}:{line_no}: expected a decimal degree, got {raw!r}")
        degrees.append(int(s))
    return np.array(degrees, dtype=np.uint64)
