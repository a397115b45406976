"""ctypes front end of the CPU oracle (``oracle/parba_oracle.c``).

TEST INFRASTRUCTURE ONLY -- the parity checker and the CPU-baseline arm of
``bench.py``.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this module; the
product package never does (``tests/test_boundary.py`` asserts that).

Every function restates the reference ``parba`` package (arXiv 1602.07106)
and cites the reference file:line it follows; parity of the restatement is
pinned against the reference's own golden vectors and against fixtures made
by running the reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libparba_oracle.so")

KIND_CRC = 0
KIND_SIMPLE = 1

MASK32 = 0xFFFFFFFF
MASK64 = 0xFFFFFFFFFFFFFFFF
DEFAULT_MULTIPLIER = 3141592653589793238  # hashing.py:32
_GOLDEN32 = 0x9E3779B9  # hashing.py:36
_GOLDEN64 = 0x9E3779B97F4A7C15  # hashing.py:37


class _Params(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64),
        ("d", ctypes.c_uint64),
        ("n0", ctypes.c_uint64),
        ("m0", ctypes.c_uint64),
        ("m", ctypes.c_uint64),
        ("kind", ctypes.c_uint32),
        ("s0", ctypes.c_uint32),
        ("s1", ctypes.c_uint32),
        ("mult", ctypes.c_uint64),
        ("seed_edges", ctypes.POINTER(ctypes.c_uint64)),
        ("W", ctypes.POINTER(ctypes.c_uint64)),
        ("flags", ctypes.c_uint32),
        ("pad", ctypes.c_uint32),
        ("max_attempts", ctypes.c_uint64),
        ("base_seed0", ctypes.c_uint64),
        ("base_seed1", ctypes.c_uint64),
        ("base_mult", ctypes.c_uint64),
    ]


def build() -> str:
    """Compile the oracle with its Makefile (gcc) if the .so is missing/stale."""
    src = os.path.join(_HERE, "parba_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "libparba_oracle.so"], check=True)
    return _LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        u64, u32, i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        P = ctypes.POINTER(_Params)
        pu64 = ctypes.c_void_p
        L.po_crc32c_u64.argtypes = [u32, u64]
        L.po_crc32c_u64.restype = u32
        L.po_h_crc.argtypes = [u64, u32, u32]
        L.po_h_crc.restype = u64
        L.po_h_simple.argtypes = [u64, u64]
        L.po_h_simple.restype = u64
        L.po_resolve_chain_block.argtypes = [P, pu64, u64, u64, pu64]
        L.po_resolve_chain_block.restype = u64
        L.po_generate_block.argtypes = [P, u64, u64, pu64]
        L.po_generate_block.restype = u64
        L.po_count_block.argtypes = [pu64, u64, pu64, u64]
        L.po_count_block.restype = None
        L.po_degree_block.argtypes = [P, u64, u64, u64, pu64]
        L.po_degree_block.restype = u64
        L.po_bb_generate.argtypes = [P, pu64]
        L.po_bb_generate.restype = None
        L.po_run_threaded.argtypes = [P, u64, u64, i32, u64, i32, u64, pu64, pu64]
        L.po_run_threaded.restype = u64
        L.po_crc32c_table.argtypes = [pu64]
        L.po_crc32c_table.restype = None
        L.po_generate_nodes.argtypes = [P, u64, u64, pu64, ctypes.POINTER(u64), ctypes.POINTER(u64)]
        L.po_generate_nodes.restype = i32
        _lib = L
    return _lib


@dataclass(frozen=True)
class OParams:
    """Graph family (generator.py:50-110 restated): uniform d, or a degree
    sequence ``degrees`` (d = None); option flags."""

    n: int
    d: int | None
    n0: int = 0
    seed_edges: tuple = ()
    kind: int = KIND_CRC
    seed0: int = 0
    seed1: int = 1
    salt: int = 0
    multiplier: int = DEFAULT_MULTIPLIER
    degrees: tuple | None = None
    no_self_loops: bool = False
    no_parallel_edges: bool = False
    max_attempts: int | None = None

    @property
    def m0(self) -> int:
        return len(self.seed_edges) // 2

    @property
    def m(self) -> int:  # generator.py:107-110
        if self.degrees is not None:
            return self.m0 + int(sum(int(x) for x in self.degrees))
        return self.m0 + (self.n - self.n0) * self.d

    def W(self) -> np.ndarray:
        """Prefix sums (degreeseq.py:109-115), n-n0+1 entries (last = m)."""
        deg = np.array(self.degrees, dtype=np.uint64)
        W = np.empty(deg.size + 1, dtype=np.uint64)
        W[0] = self.m0
        np.cumsum(deg, out=W[1:])
        W[1:] += np.uint64(self.m0)
        return W

    @property
    def flags(self) -> int:
        return (1 if self.no_self_loops else 0) | (2 if self.no_parallel_edges else 0)

    def crc_seeds(self) -> tuple[int, int]:  # hashing.py:73-77
        return (self.seed0 + self.salt) & MASK32, (self.seed1 + self.salt * _GOLDEN32) & MASK32

    def simple_multiplier(self) -> int:  # hashing.py:79-85
        return (self.multiplier + 2 * self.salt * _GOLDEN64) & MASK64

    def _c(self):
        seed = np.ascontiguousarray(np.array(self.seed_edges, dtype=np.uint64))
        s0, s1 = self.crc_seeds()
        W = self.W() if self.degrees is not None else None
        st = _Params(self.n, self.d or 0, self.n0, self.m0, self.m, self.kind, s0, s1,
                     self.simple_multiplier(),
                     seed.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)) if seed.size else None,
                     W.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)) if W is not None else None,
                     self.flags, 0, self.max_attempts or 0, self.seed0 & MASK64, self.seed1 & MASK64,
                     self.multiplier & MASK64)
        return st, (seed, W)  # keep the arrays alive alongside the struct


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def crc32c_u64(seed: int, word: int) -> int:
    return int(lib().po_crc32c_u64(seed & MASK32, word & MASK64))


def crc32c_table() -> np.ndarray:
    out = np.zeros(256, dtype=np.uint32)
    lib().po_crc32c_table(_ptr(out))
    return out


def h_crc(r: int, s0: int = 0, s1: int = 1) -> int:
    assert r >= 1
    return int(lib().po_h_crc(r, s0, s1))


def h_simple(r: int, mult: int = DEFAULT_MULTIPLIER) -> int:
    assert r >= 1
    return int(lib().po_h_simple(r, mult))


def hash_many(p: OParams, r: np.ndarray) -> np.ndarray:
    r = np.asarray(r, dtype=np.uint64)
    if p.kind == KIND_CRC:
        s0, s1 = p.crc_seeds()
        return np.array([lib().po_h_crc(int(x), s0, s1) for x in r], dtype=np.uint64)
    m = p.simple_multiplier()
    return np.array([lib().po_h_simple(int(x), m) for x in r], dtype=np.uint64)


def resolve_chain_block(p: OParams, r0: np.ndarray, stop_below: int) -> tuple[np.ndarray, int]:
    r0 = np.ascontiguousarray(r0, dtype=np.uint64)
    out = np.empty_like(r0)
    st, _keep = p._c()
    probes = lib().po_resolve_chain_block(ctypes.byref(st), _ptr(r0), r0.size, stop_below, _ptr(out))
    return out, int(probes)


class NotNodeBoundary(ValueError):
    pass


class Infeasible(RuntimeError):
    def __init__(self, edge: int):
        super().__init__(f"edge {edge}: no fresh target")
        self.edge = edge


def generate_block(p: OParams, lo: int, hi: int) -> tuple[np.ndarray, int]:
    """generate_block (generator.py:258-325); flag modes are node-granular
    (raise NotNodeBoundary / Infeasible like the reference's errors)."""
    out = np.empty((hi - lo, 2), dtype=np.uint64)
    st, _keep = p._c()
    if p.flags:
        probes, fail = ctypes.c_uint64(0), ctypes.c_uint64(0)
        rc = lib().po_generate_nodes(ctypes.byref(st), lo, hi, _ptr(out), ctypes.byref(probes), ctypes.byref(fail))
        if rc == 1:
            raise NotNodeBoundary(f"[{lo}, {hi}) is not node-aligned")
        if rc == 2:
            raise Infeasible(int(fail.value))
        return out, int(probes.value)
    probes = lib().po_generate_block(ctypes.byref(st), lo, hi, _ptr(out))
    return out, int(probes)


def count_block(counts: np.ndarray, edges: np.ndarray) -> None:
    edges = np.ascontiguousarray(edges, dtype=np.uint64)
    assert counts.dtype == np.int64 and counts.flags.c_contiguous
    lib().po_count_block(_ptr(edges), edges.size // 2, _ptr(counts), counts.size)


def degree_block(p: OParams, lo: int, hi: int, K: int, counts: np.ndarray | None = None):
    if counts is None:
        counts = np.zeros(K, dtype=np.int64)
    st, _keep = p._c()
    probes = lib().po_degree_block(ctypes.byref(st), lo, hi, K, _ptr(counts))
    return counts, int(probes)


def bb_generate(p: OParams) -> np.ndarray:
    e = np.empty(2 * p.m, dtype=np.uint64)
    st, _keep = p._c()
    lib().po_bb_generate(ctypes.byref(st), _ptr(e))
    return e


MODE_STORE, MODE_WINDOW, MODE_DISCARD = 0, 1, 2


def run_threaded(p: OParams, lo: int, hi: int, mode: int, K: int = 0, threads: int = 1,
                 batch: int = 1 << 16, out: np.ndarray | None = None):
    """Threaded reference driver (driver.py:161-270): returns (out|counts, probes)."""
    st, _keep = p._c()
    counts = np.zeros(max(K, 1), dtype=np.int64) if mode == MODE_WINDOW else None
    if mode == MODE_STORE and out is None:
        out = np.empty((hi - lo, 2), dtype=np.uint64)
    probes = lib().po_run_threaded(ctypes.byref(st), lo, hi, mode, K, threads, batch,
                                   _ptr(out) if out is not None else None,
                                   _ptr(counts) if counts is not None else None)
    if mode == MODE_WINDOW:
        return counts[:K], int(probes)
    return out, int(probes)
