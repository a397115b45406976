"""End-to-end host-array throughput: generate_block(lo, lo + N, C2) into a
fresh host array under several pipeline settings (environment knobs of
parba_host.cu: PARBA_HOST_PAIRS, PARBA_E2E_CHUNK_LOG2, PARBA_E2E_SLOTS,
PARBA_E2E_ROWS_FRAC, PARBA_HOST_THREADS).  Each setting runs in a fresh
process (the library reads the knobs per call, but staging is cached).
Prints one JSON line per setting.

    python tools/e2e_perf.py [--edges N] SETTING...   (SETTING = "K=V,K=V" or "default")
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(edges: int, reps: int = 3) -> float:
    sys.path.insert(0, ROOT)
    import paper_1602_07106_b200 as pb

    p = pb.GenParams(n=10**8, d=10)
    best = 1e9
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        arr, _ = pb.generate_block(0, edges, p)
        best = min(best, time.perf_counter() - t0)
        del arr
    return edges / best


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--edges", type=int, default=250_000_000)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--repeat", type=int, default=2, help="processes per setting")
    ap.add_argument("settings", nargs="*", default=["default"])
    a = ap.parse_args()
    if a.child:
        print(child(a.edges))
        sys.exit(0)
    for s in [x for x in a.settings for _ in range(a.repeat)]:
        env = dict(os.environ)
        if s != "default":
            env.update(kv.split("=", 1) for kv in s.split(","))
        out = subprocess.run([sys.executable, __file__, "--child", "--edges", str(a.edges)], env=env,
                             capture_output=True, text=True)
        val = float(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else None
        print(json.dumps({"setting": s, "edges_per_s": val, "err": out.stderr[-300:] if val is None else ""}),
              flush=True)
