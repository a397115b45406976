"""Position-hash families (reference: parba/hashing.py).

``HashConfig`` / ``HashKind`` are the reference's configuration objects
(hashing.py:43-85) with the same validation and salt folding.  Evaluating a
hash (``h_crc``, ``h_simple``, ``hash_value``, ``hash_many``) runs the CUDA
kernel ``parba_hash`` -- the same device code the generator uses -- so there is
exactly one implementation of h on this path and no CPU fallback.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .errors import ParameterError

MASK32 = 0xFFFFFFFF
MASK64 = 0xFFFFFFFFFFFFFFFF

# hashing.py:32 -- default SIMPLE multiplier (first 19 digits of pi; even,
# see SURVEY Appendix A.1: the reference does not enforce oddness).
DEFAULT_MULTIPLIER = 3141592653589793238
_GOLDEN32 = 0x9E3779B9  # hashing.py:36
_GOLDEN64 = 0x9E3779B97F4A7C15  # hashing.py:37


class HashKind(enum.Enum):
    CRC = "crc"
    SIMPLE = "simple"


@dataclass(frozen=True)
class HashConfig:
    """The position-hash family (hashing.py:48-85): kind, CRC seeds (used as
    32-bit values), rejection-attempt salt and SIMPLE multiplier."""

    kind: HashKind = HashKind.CRC
    seed0: int = 0
    seed1: int = 1
    attempt_salt: int = 0
    multiplier: int = DEFAULT_MULTIPLIER

    def __post_init__(self) -> None:
        for name in ("seed0", "seed1", "attempt_salt", "multiplier"):
            v = getattr(self, name)
            if not 0 <= v <= MASK64:
                raise ParameterError(f"{name} must be an unsigned 64-bit value, got {v}")

    def with_attempt(self, salt: int) -> "HashConfig":
        return replace(self, attempt_salt=salt)

    def crc_seeds(self) -> tuple[int, int]:
        """Effective 32-bit seeds, salt folded in (hashing.py:73-77)."""
        return (self.seed0 + self.attempt_salt) & MASK32, (self.seed1 + self.attempt_salt * _GOLDEN32) & MASK32

    def simple_multiplier(self) -> int:
        """Effective multiplier, salt folded in with an even offset (hashing.py:79-85)."""
        return (self.multiplier + 2 * self.attempt_salt * _GOLDEN64) & MASK64


def c_params(cfg: HashConfig, n: int = 1, d: int = 1, n0: int = 0, m0: int = 0,
             seed_ptr: int | None = None) -> _lib.CParams:
    """parba_params_t for a family (a 1-node dummy graph when only h is needed).
    The base seeds / multiplier feed the retry families of no_parallel_edges
    (HashConfig.with_attempt: attempt a >= 1 replaces the salt by a)."""
    s0, s1 = cfg.crc_seeds()
    p = _lib.CParams(n, d, n0, m0, m0 + (n - n0) * d,
                     _lib.HASH_CRC if cfg.kind is HashKind.CRC else _lib.HASH_SIMPLE,
                     s0, s1, 0, cfg.simple_multiplier(), seed_ptr)
    p.base_seed0 = cfg.seed0 & MASK32
    p.base_seed1 = cfg.seed1 & MASK32
    p.base_mult = cfg.multiplier & MASK64
    return p


def hash_many(r, cfg: HashConfig, device=None) -> np.ndarray:
    """Elementwise h(r) on the GPU (hashing.py:194-198); every r >= 1."""
    r = np.ascontiguousarray(np.asarray(r, dtype=np.uint64)).reshape(-1)
    if r.size and int(r.min()) < 1:
        raise ParameterError(f"hash argument must be >= 1, got {int(r.min())}")
    torch = _lib.torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if r.size == 0:
        return np.empty(0, dtype=np.uint64)
    rd = _lib.to_device_u64(torch, r, dev)
    out = torch.empty_like(rd)
    L = _lib.load()
    with torch.cuda.device(dev):
        p = c_params(cfg)
        _lib.check(L.parba_hash(p, rd.data_ptr(), r.size, out.data_ptr(), _lib.stream_ptr(torch, dev)))
        return out.cpu().numpy().view(np.uint64)


def _scalar(r: int, cfg: HashConfig) -> int:
    if r < 1:
        raise ParameterError(f"hash argument must be >= 1, got {r}")
    if r > MASK64:
        raise ParameterError(f"hash argument must fit 64 bits, got {r}")
    return int(hash_many(np.array([r], dtype=np.uint64), cfg)[0])


def h_crc(r: int, cfg: HashConfig) -> int:
    """((crc(s0,r)<<32) + crc(s1,r)) % r (hashing.py:119-125), on the GPU."""
    return _scalar(r, replace(cfg, kind=HashKind.CRC))


def h_simple(r: int, cfg: HashConfig) -> int:
    """umulhi((r*M) mod 2^64, r) (hashing.py:128-138), on the GPU."""
    return _scalar(r, replace(cfg, kind=HashKind.SIMPLE))


def hash_value(r: int, cfg: HashConfig) -> int:
    return _scalar(r, cfg)


# ---------------------------------------------------------------------------
# The CRC32-C primitive and the vectorized helpers of hashing.py:88-198.

_CRC32C_POLY = 0x82F63B78  # hashing.py:40


def _build_crc32c_table() -> tuple[int, ...]:
    """The 256-entry reflected table (hashing.py:88-95): a constant of the
    hash family, built once on the host; every CRC evaluation runs on the GPU."""
    table = []
    for i in range(256):
        c = i
        for _ in range(8):
            c = (c >> 1) ^ _CRC32C_POLY if c & 1 else c >> 1
        table.append(c)
    return tuple(table)


CRC32C_TABLE: tuple[int, ...] = _build_crc32c_table()


def _dev_u64(a):
    torch = _lib.torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    return torch, dev, _lib.to_device_u64(torch, a, dev)


def crc32c_u64_many(seed: int, words) -> np.ndarray:
    """Elementwise crc32c_u64(seed, w) (hashing.py:158-165), on the GPU."""
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint64)).reshape(-1)
    if w.size == 0:
        return np.zeros(0, dtype=np.uint64)
    torch, dev, wd = _dev_u64(w)
    out = torch.empty_like(wd)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().parba_crc32c(seed & MASK32, wd.data_ptr(), w.size, out.data_ptr(),
                                            _lib.stream_ptr(torch, dev)))
        return out.cpu().numpy().view(np.uint64)


def crc32c_u64(seed: int, word: int) -> int:
    """CRC32-C of one little-endian 64-bit word on `seed`, raw (no
    inversion): _mm_crc32_u64 semantics (hashing.py:105-116)."""
    return int(crc32c_u64_many(seed, np.array([word & MASK64], dtype=np.uint64))[0])


def mulhi_u64(a, b) -> np.ndarray:
    """High 64 bits of the elementwise 128-bit product (hashing.py:168-176)."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64)).reshape(-1)
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint64)).reshape(-1)
    if a.shape != b.shape:
        raise ParameterError("mulhi_u64 operands must have the same shape")
    if a.size == 0:
        return np.zeros(0, dtype=np.uint64)
    torch, dev, ad = _dev_u64(a)
    bd = _lib.to_device_u64(torch, b, dev)
    out = torch.empty_like(ad)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().parba_mulhi_u64(ad.data_ptr(), bd.data_ptr(), a.size, out.data_ptr(),
                                               _lib.stream_ptr(torch, dev)))
        return out.cpu().numpy().view(np.uint64)


def h_crc_many(r, cfg: HashConfig) -> np.ndarray:
    """Elementwise h_crc (hashing.py:179-184); every r >= 1."""
    return hash_many(r, replace(cfg, kind=HashKind.CRC))


def h_simple_many(r, cfg: HashConfig) -> np.ndarray:
    """Elementwise h_simple (hashing.py:187-191); every r >= 1."""
    return hash_many(r, replace(cfg, kind=HashKind.SIMPLE))
