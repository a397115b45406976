"""``bb_generate`` / ``edge_list`` names of the reference (oracle.py:45-112).

The reference's sequential Batagelj-Brandes fill E[2i+1] = E[h(2i+1)] is, by
the paper's equivalence, entry-for-entry the same array as
the independent chain recomputation.  So the derandomized array is produced
here by the GPU store kernel (seed prefix + generate_block over [m0, m)); the
rng mode has no derandomized counterpart and is not on the B200 path.
This module is NOT the parity oracle -- that lives in oracle/ (tests only).
"""

from __future__ import annotations

import numpy as np

from .errors import ParameterError
from .generator import GenParams, generate_block

DEFAULT_CAP = 10**8  # oracle.py:29


def bb_generate(p: GenParams, mode: str = "derandomized", rng_seed: int = 0, cap: int = DEFAULT_CAP,
                engine: str = "auto") -> np.ndarray:
    if p.no_self_loops or p.no_parallel_edges:
        raise ParameterError("the sequential oracle supports plain mode only")
    if mode not in ("derandomized", "rng"):
        raise ParameterError(f"unknown mode {mode!r}")
    if mode == "rng":
        raise ParameterError("rng mode draws from a host PRNG stream; it is not on the B200 path")
    if engine not in ("auto", "python", "compiled"):
        raise ParameterError(f"unknown engine {engine!r}")
    if p.m > cap:
        raise ParameterError(f"m = {p.m} exceeds the oracle cap {cap}")
    e = np.empty(2 * p.m, dtype=np.uint64)
    e[: 2 * p.m0] = p.seed_edges
    blk, _ = generate_block(p.m0, p.m, p)
    e[2 * p.m0:] = blk.reshape(-1)
    return e


def edge_list(e: np.ndarray, m0: int = 0) -> np.ndarray:
    return e[2 * m0:].reshape(-1, 2)
