"""Practical ceiling for the 16384^2 dense activity scan's traffic (33.5 MB
read + up to 33.5 MB written): CUDA-graph replays of 20 back-to-back
torch copies / fills / 4-byte memsets over 4 L2-cold buffer sets, beside
the scan itself (tools/scan_time.py).  python tools/scan_ceiling.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def graph_us(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3):
            fn(i)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * reps)


def main():
    nb = 16384 * 16384 // 8  # one bit plane, bytes
    src = [torch.ones(nb // 4, dtype=torch.int32, device="cuda") for _ in range(4)]
    dst = [torch.empty_like(x) for x in src]
    cnt = torch.zeros(64, dtype=torch.int32, device="cuda")
    peak = 6531.9
    rows = {
        "copy 33.5MB->33.5MB": (graph_us(lambda i: dst[i % 4].copy_(src[i % 4])), 2 * nb),
        "fill 33.5MB": (graph_us(lambda i: dst[i % 4].zero_()), nb),
        "read-reduce 33.5MB (amax)": (graph_us(lambda i: torch.amax(src[i % 4], dim=0, out=cnt[0])), nb),
        "memset 4 B": (graph_us(lambda i: cnt[i % 4 : i % 4 + 1].zero_()), 0),
    }
    for k, (us, b) in rows.items():
        print(f"{k:28s} {us:7.2f} us  {b / us / 1e3:7.0f} GB/s  {b / us / 1e3 / peak:.2f}")


if __name__ == "__main__":
    main()
