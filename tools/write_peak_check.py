import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import torch
import paper_1602_07106_b200 as pb
L = pb._lib.load()
dev = torch.device("cuda", 0)
out = torch.empty(2 * 10**9, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream(dev)
for rep in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    pb._lib.check(L.parba_peak_write(out.data_ptr(), 16 * 10**9, st.cuda_stream))
    e1.record(st)
    e1.synchronize()
    print("write GB/s", 16e9 / (e0.elapsed_time(e1) / 1e3) / 1e9)
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); out.fill_(7); e1.record(st); e1.synchronize()
    print("torch fill GB/s", 16e9 / (e0.elapsed_time(e1) / 1e3) / 1e9)
