"""Binary edge-file writer (f2) throughput: write_edges_binary of an
n=1e8/d=2 graph (2e8 edges, 3.2 GB) to /dev/shm (tmpfs) and to /tmp, wall
clock including the file's creation and close.  Prints JSON."""
import json
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1602_07106_b200 as pb
from paper_1602_07106_b200 import io as pio

p = pb.GenParams(n=10**8, d=2)
res = {"edges": p.m, "bytes": 16 * p.m}
mode = os.environ.get("PARBA_WRITER_PWRITE", "0")
res["path"] = "pinned buffers + one pwrite thread" if mode == "1" else "parba_write_binary (mapped range, host pipeline)"
for name, d in (("dev_shm", "/dev/shm"), ("tmp", "/tmp")):
    free = shutil.disk_usage(d).free
    if free < 2 * 16 * p.m:
        res[name] = f"skipped: {free / 1e9:.1f} GB free"
        continue
    path = os.path.join(d, "parba_writer_perf.bin")
    pio.write_edges_binary(path, pb.GenParams(n=1000, d=2))  # warm the path
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nbytes, _ = pio.write_edges_binary(path, p)
    t = time.perf_counter() - t0
    os.remove(path)
    res[name] = {"s": t, "edges_per_s": p.m / t, "GB_per_s": nbytes / t / 1e9}
print(json.dumps(res))
