import sys, os, ctypes as C, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2502_18738_b200 as F
from paper_2502_18738_b200 import _lib as L, synthetic as S
n = 16384
b = F.FireBatch((n, n), 1, max_steps=8)
b.reset(S.random_blocks(n, n, 8, 5, seed=3))
st = b.struct()
for name in ("scan",):
    ts = []
    for _ in range(30):
        b.list_count.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); L.check(L.lib().fc_activity_scan(C.byref(b.grid), C.byref(st), 0, L.stream_ptr()), "x"); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(name, "us", 1e3*np.mean(ts[5:]), "GB/s", 67.2e6/(np.mean(ts[5:])/1e3)/1e9)
