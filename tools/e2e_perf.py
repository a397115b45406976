"""End-to-end host-array throughput: generate_block(lo, lo + N, C2) into a
fresh host array, targets-only pipeline vs 16-byte rows (PARBA_HOST_PAIRS=1),
for several host-thread counts.  Prints JSON lines.

    python tools/e2e_perf.py [--edges N] [--threads 4,8,16]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1602_07106_b200 as pb  # noqa: E402


def rate(p, lo, n, reps=3):
    best = 1e9
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        arr, _ = pb.generate_block(lo, lo + n, p)
        dt = time.perf_counter() - t0
        del arr
        best = min(best, dt)
    return n / best


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--edges", type=int, default=250_000_000)
    ap.add_argument("--threads", default="")
    a = ap.parse_args()
    p = pb.GenParams(n=10**8, d=10)
    out = {"edges": a.edges}
    os.environ["PARBA_HOST_PAIRS"] = "1"
    out["pairs"] = rate(p, 0, a.edges)
    del os.environ["PARBA_HOST_PAIRS"]
    for t in [x for x in a.threads.split(",") if x] or [""]:
        if t:
            os.environ["PARBA_HOST_THREADS"] = t
        out[f"targets_t{t or 'all'}"] = rate(p, 0, a.edges)
    print(json.dumps(out), flush=True)
