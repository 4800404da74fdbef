"""Where the e2e (host buffers) time of the c1 ensemble call goes: CUDA
events around each phase of EnsembleRunner's work.  python tools/e2e_breakdown.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402
from paper_2502_18738_b200.ensemble import EnsembleRunner  # noqa: E402


def main():
    H = 2048
    env = S.make_environment(H, seed=1)
    env_host = torch.stack([torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)) for a in
                            (env.elevation, env.wind_speed, env.wind_direction, env.canopy,
                             env.density)]).pin_memory()
    init_host = torch.from_numpy(S.center_ignition(H).astype(np.uint8)).pin_memory()
    ph = S.ensemble_ph(16)
    params = [(0.045, 0.131, 0.078, float(p), 0.3) for p in ph]
    r = EnsembleRunner((H, H), 16, 500)
    for _ in range(2):
        r(env_host, init_host, params, list(range(16)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        r(env_host, init_host, params, list(range(16)))
    print("e2e call ms", (time.perf_counter() - t0) / 5 * 1e3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prev = None
    for _ in range(10):
        t = r.submit(env_host, init_host, params, list(range(16)))
        if prev is not None:
            prev.result()
        prev = t
    prev.result()
    print("e2e pipelined ms per call", (time.perf_counter() - t0) / 10 * 1e3)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    r = r.slots[0]
    b = r.batch
    for rep in range(2):
        torch.cuda.synchronize()
        ev[0].record()
        r.env_dev.copy_(env_host, non_blocking=True)
        r.init_dev.copy_(init_host, non_blocking=True)
        ev[1].record()
        e = r.env_dev
        land = F.DeviceLandscape.from_elevation(e[0], e[1], e[2], e[3], e[4])
        ev[2].record()
        b.reset(r.init_dev)
        ev[3].record()
        b.run(land, 500)
        ev[4].record()
        bu, bd = b.unpack()
        ev[5].record()
        r.out_b.copy_(bu, non_blocking=True)
        r.out_d.copy_(bd, non_blocking=True)
        ev[6].record()
        r.out_acc.copy_(b.acc, non_blocking=True)
        ev[7].record()
        torch.cuda.synchronize()
    names = ["h2d env+init", "landscape build", "reset", "run", "unpack", "d2h states",
             "d2h acc"]
    for i, n in enumerate(names):
        print(f"{n:16s} {ev[i].elapsed_time(ev[i + 1]):8.3f} ms")


if __name__ == "__main__":
    main()
