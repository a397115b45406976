import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1602_07106_b200 as pb
from paper_1602_07106_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10**7
rng = np.random.default_rng(0)
deg = np.minimum(rng.zipf(2.0, size=n) + 7, 10_000).astype(np.uint64)
deg[rng.random(n) < 0.05] = 0
deg[0] = 10
p = pb.GenParams(n=n, degrees=deg)
dev = torch.device("cuda", 0)
cp = p._device_params(dev)
L = _lib.load()
out = torch.empty(2 * p.m, dtype=torch.int64, device=dev)
prb = torch.zeros(1, dtype=torch.int64, device=dev)
for _ in range(2):
    _lib.check(L.parba_generate(cp, 0, p.m, out.data_ptr(), prb.data_ptr(), torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("ok", p.m)
