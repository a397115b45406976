"""Kernel seam of the reference (parba/_kernels.py): ``resolve_chain_block``
and ``warmup`` under the reference's module path, so code that imports
``parba._kernels`` directly finds them here.  The chains run in the CUDA
library; ``warmup`` loads it and initialises the device ahead of use
(the reference compiles its numba kernels before forking, _kernels.py:138-143)."""

from __future__ import annotations

import numpy as np

from .generator import resolve_chain_block
from .hashing import HashConfig, HashKind

__all__ = ["resolve_chain_block", "warmup"]


def warmup() -> None:
    r = np.array([1, 9, 11], dtype=np.uint64)
    resolve_chain_block(r, 0, HashConfig(kind=HashKind.SIMPLE))
    resolve_chain_block(r, 0, HashConfig(kind=HashKind.CRC))
