"""Spread of per-warp completion times of one C2 store launch (diagnostic
build: -DPARBA_WARP_TIMES=1).  python tools/warp_times.py build_ab/lib_wt.so"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1602_07106_b200 import _lib, hashing

L = _lib.load(sys.argv[1])
dev = torch.device("cuda", 0)
p = hashing.c_params(hashing.HashConfig(), n=10**8, d=10)
out = torch.empty(2 * 10**9, dtype=torch.int64, device=dev)
prb = torch.zeros(1, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.check(L.parba_generate(p, 0, 10**9, out.data_ptr(), prb.data_ptr(), st))
torch.cuda.synchronize()
nw = 148 * 32
t = np.zeros(2 * nw, dtype=np.uint64)
fn = L.parba_debug_warp_times
fn.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
_lib.check(fn(t.ctypes.data, nw))
start, end = t[0::2].astype(np.int64), t[1::2].astype(np.int64)
t0 = start.min()
s, e = (start - t0) / 1e3, (end - t0) / 1e3
print(f"kernel span {e.max():.1f} us; warp end: min {e.min():.1f} p10 {np.percentile(e,10):.1f} "
      f"median {np.median(e):.1f} p90 {np.percentile(e,90):.1f} max {e.max():.1f}; start max {s.max():.1f}")
print(f"avg busy fraction {np.mean(e - s) / e.max():.4f}")
by_wib = (e.reshape(148, 32)).mean(axis=0)
print("mean end by warp-in-block:", " ".join(f"{x:.0f}" for x in by_wib))
