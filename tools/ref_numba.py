"""Time the reference's own CPU path (parba, numba, installed under
baseline/_ref) on this host's cores: store mode (generate_block per 2^16
batch, the reference driver's batch size) and the degree window, on
contiguous sub-ranges at the top of a config's edge-ID space, forked over
all host cores as the reference's driver.run does.  Prints JSON.

    python tools/ref_numba.py [--edges N] [--mode store|window|full]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import reference_numba  # noqa: E402

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--edges", type=int, default=None)
    ap.add_argument("--mode", default="store")
    ap.add_argument("--budget", type=float, default=8.0)
    a = ap.parse_args()
    t0 = time.perf_counter()
    print(json.dumps(reference_numba(a.mode, sample_edges=a.edges, budget_s=a.budget)), flush=True)
    print(f"wall {time.perf_counter() - t0:.1f}s", file=sys.stderr)
