"""(Record of a dropped experiment: the PARBA_SCATTER2 knob is not in the shipped
library; see profiles/r02_ab_c4_scatter_lean.txt.)
A/B of the full-histogram scatter (C4 and two other shapes): libraries
given on the command line, and for the current one the env knob
PARBA_SCATTER2 (1: lean scatter, 0: first form).  Counts checked equal to
the direct-atomic kernel.  CUDA-event timed, median of 5."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1602_07106_b200 as pb
from paper_1602_07106_b200 import _lib

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev).cuda_stream
libs = sys.argv[1:] or [None]
shapes = (("C4", dict(n=10**8, d=16)), ("n2e8_d8", dict(n=2 * 10**8, d=8)), ("n5e7_d32", dict(n=5 * 10**7, d=32)))
refs = {}
for path in libs:
    _lib._lib = None
    L = _lib.load(path) if path else _lib.load()
    for knob in ("1", "0"):
        os.environ["PARBA_SCATTER2"] = knob
        for name, kw in shapes:
            p = pb.GenParams(**kw)
            cp = p._device_params(dev)
            prb = torch.zeros(1, dtype=torch.int64, device=dev)
            c = torch.zeros(p.n, dtype=torch.int32, device=dev)
            if name not in refs:
                os.environ["PARBA_FULL_MODE"] = "direct"
                _lib.check(L.parba_degree_full(cp, 0, p.m, c.data_ptr(), prb.data_ptr(), st))
                torch.cuda.synchronize()
                refs[name] = c.clone()
                os.environ.pop("PARBA_FULL_MODE")
            c.zero_()
            _lib.check(L.parba_degree_full(cp, 0, p.m, c.data_ptr(), prb.data_ptr(), st))
            torch.cuda.synchronize()
            ok = torch.equal(refs[name], c)
            ts = []
            for _ in range(5):
                c.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _lib.check(L.parba_degree_full(cp, 0, p.m, c.data_ptr(), prb.data_ptr(), st))
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[2]
            print(f"{os.path.basename(path or 'in-tree')} scatter2={knob} {name} ms={ms:.3f} "
                  f"edges/s={p.m / ms * 1e3:.4e} equal={ok}", flush=True)
            del c
