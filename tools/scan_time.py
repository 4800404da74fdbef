"""Dense activity scan (fc_activity_scan) of the config-3 domain: per-scan
time, event-timed alone and as 20 back-to-back launches in one CUDA graph;
algorithmic bytes = burning plane read + zero next state of quiet tiles.
FIRECELL_SO=<build> python tools/scan_time.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import _lib as L, synthetic as S  # noqa: E402


def main():
    n = 16384
    # four states scanned in turn: each scan's 67 MB of plane traffic is
    # evicted from the 126 MB L2 by the next three before it comes round
    bs = []
    for k in range(4):
        b = F.FireBatch((n, n), 1, max_steps=8)
        b.reset(S.random_blocks(n, n, 8, 5, seed=3 + k))
        bs.append((b, b.struct()))
    b, st = bs[0]
    it = [0]

    def scan():
        bb, ss = bs[it[0] % 4]
        it[0] += 1
        L.check(L.lib().fc_activity_scan(C.byref(bb.grid), C.byref(ss), 0, L.stream_ptr()),
                "scan")
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        scan()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    live = int(b.list_count[0].item())
    tiles = n * n // 1024
    byts = 128.0 * tiles + 128.0 * (tiles - live)
    one = np.mean(ts[5:]) * 1e3
    g = F.CapturedSequence(lambda: [scan() for _ in range(20)])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    per = e0.elapsed_time(e1) * 1e3 / 100
    peak = 6531.9
    print(f"{os.environ.get('FIRECELL_SO', 'default')}: alone {one:.1f} us "
          f"({byts / one / 1e3:.0f} GB/s, {byts / one / 1e3 / peak:.2f}); in graph {per:.1f} us "
          f"({byts / per / 1e3:.0f} GB/s, {byts / per / 1e3 / peak:.2f}); live {live}")


if __name__ == "__main__":
    main()
