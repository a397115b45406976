import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as O
from paper_1602_07106_b200 import _lib, hashing
for lib in sys.argv[1:]:
    L = _lib.load(lib); _lib._lib = None
    ok = True
    for (n, d, lo, hi) in ((10**5, 4, 0, 4*10**5), (10**8, 10, 123457, 123457 + 2*10**6), (10**8, 10, 9*10**8 + 5, 9*10**8 + 2*10**6 + 77), (2**40, 7, 2**40, 2**40 + 300001), (10**9, 3, 2**30 + 1000, 2**30 + 2*10**6 + 3), (10**9, 100, 5*10**10+3, 5*10**10+1000003)):
        p = hashing.c_params(hashing.HashConfig(), n=n, d=d)
        out = torch.empty(2*(hi-lo), dtype=torch.int64, device="cuda"); prb = torch.zeros(1, dtype=torch.int64, device="cuda")
        _lib.check(L.parba_generate(p, lo, hi, out.data_ptr(), prb.data_ptr(), torch.cuda.current_stream().cuda_stream))
        got = out.cpu().numpy().view(np.uint64).reshape(-1, 2)
        want, wp = O.generate_block(O.OParams(n=n, d=d), lo, hi)
        ok &= bool(np.array_equal(got, want)) and int(prb.item()) == wp
    print(os.path.basename(lib), "parity", ok)
