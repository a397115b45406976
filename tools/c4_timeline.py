"""In-situ kernel timeline of one C4 full-histogram step (n=1e8, d=16) from
torch.profiler (CUPTI): start, duration and the idle gap before every kernel
of the last of three steps.  python tools/c4_timeline.py [LIB]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_1602_07106_b200 import _lib, hashing

L = _lib.load(sys.argv[1]) if len(sys.argv) > 1 else _lib.load()
p = hashing.c_params(hashing.HashConfig(), n=10**8, d=16)
c = torch.zeros(10**8, dtype=torch.int32, device="cuda")
prb = torch.zeros(1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def step():
    c.zero_()
    _lib.check(L.parba_degree_full(p, 0, 16 * 10**8, c.data_ptr(), prb.data_ptr(), st))


for _ in range(2):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
            key=lambda e: e.time_range.start)
t_end_prev = None
rows = []
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = 0 if t_end_prev is None else s - t_end_prev
    rows.append((e.name[:70], s, d, gap))
    t_end_prev = e.time_range.end
# the last step: from the last FillFunctor (c.zero_()) on
idx = [i for i, r in enumerate(rows) if "FillFunctor" in r[0] or "emset" in r[0]]
if not idx:  # no fill event recorded: split the events into the three steps evenly
    idx = [len(rows) * 2 // 3]
last = rows[idx[-1]:]
tot = last[-1][1] + last[-1][2] - last[0][1]
print(f"last step: {tot / 1000:.3f} ms wall, kernels {sum(r[2] for r in last) / 1000:.3f} ms, "
      f"gaps {sum(r[3] for r in last[1:]) / 1000:.3f} ms")
for name, s, d, gap in last:
    print(f"{(s - last[0][1]) / 1000:9.3f} ms  dur {d / 1000:8.3f} ms  gap {gap / 1000:7.3f} ms  {name}")
