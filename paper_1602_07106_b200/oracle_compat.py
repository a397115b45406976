"""``bb_generate`` / ``edge_list`` of the reference (oracle.py:45-112).

The reference's bb_generate is its sequential Batagelj-Brandes fill -- E[2i]
= source(i), E[2i+1] = E[x] with x = h(2i+1) -- used as ground truth for its
parallel chain recomputation (the verify command, cli.py:332-351).  Here the
same array is built on the device AS AN ARRAY (C ABI ``parba_bb_fill``): one
hash per edge gives each odd cell a pointer, pointer jumping resolves the
pointers to source or seed cells, and the odd cells are gathered -- no hash
chain is run, so comparing it with ``generate_block`` (the tile kernels'
chain recomputation) is an independent check, as in the reference.

``engine`` keeps the reference's values: "python" and "compiled" name the
reference's two fills (identical arrays); both select the device fill here,
and "compiled" keeps the reference's uniform-degree restriction.  rng mode
draws from a host PCG64 stream and is not on the B200 path.
This module is NOT the parity oracle -- that lives in oracle/ (tests only).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ParameterError
from .generator import GenParams, _device

DEFAULT_CAP = 10**8  # oracle.py:29


def bb_generate(p: GenParams, mode: str = "derandomized", rng_seed: int = 0, cap: int = DEFAULT_CAP,
                engine: str = "auto", device=None) -> np.ndarray:
    """The full edge array E[0 .. 2m) (uint64), seed cells included."""
    if p.no_self_loops or p.no_parallel_edges:
        raise ParameterError("the sequential oracle supports plain mode only")
    if mode not in ("derandomized", "rng"):
        raise ParameterError(f"unknown mode {mode!r}")
    if p.m > cap:
        raise ParameterError(f"m = {p.m} exceeds the oracle cap {cap}")
    if mode == "rng":
        raise ParameterError("rng mode draws from a host PRNG stream; it is not on the B200 path")
    if engine not in ("auto", "python", "compiled"):
        raise ParameterError(f"unknown engine {engine!r}")
    if engine == "compiled" and p.d is None:
        raise ParameterError("the compiled fill supports uniform degrees only")
    torch, dev = _device(device)
    E = torch.empty(max(2 * p.m, 1), dtype=torch.int64, device=dev)
    link = torch.empty(max(p.m - p.m0, 1), dtype=torch.int64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    passes = ctypes.c_int(0)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().parba_bb_fill(p._device_params(dev), E.data_ptr(), link.data_ptr(), flag.data_ptr(),
                                             ctypes.byref(passes), _lib.stream_ptr(torch, dev)))
        return E[: 2 * p.m].cpu().numpy().view(np.uint64)


def edge_list(e: np.ndarray, m0: int = 0) -> np.ndarray:
    """The generated region of an edge array as (m - m0, 2) pairs."""
    return e[2 * m0:].reshape(-1, 2)
