"""Per-launch device time of the c1 workload at M members (CUDA events
around each 8-step fc_run), plus the reset:  MS=1,16 python tools/launch_times.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402


def main():
    env = S.make_environment(2048, seed=1)
    dl = F.DeviceLandscape.from_environment(env)
    init = torch.as_tensor(S.center_ignition(2048).astype(np.uint8), device="cuda")
    win = int(os.environ.get("WINDOW", 8))
    for M in [int(x) for x in os.environ.get("MS", "1,16").split(",")]:
        b = F.FireBatch((2048, 2048), M, max_steps=500)
        ph = S.ensemble_ph(M)
        b.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, p, 0.3) for p in ph]))
        b.set_seeds(list(range(M)))
        for rep in range(2):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 + 500 // win + 1)]
            ev[0].record()
            b.reset(init)
            ev[1].record()
            n = 0
            for a in range(0, 500, win):
                b.run(dl, min(win, 500 - a), window=win)
                n += 1
                ev[1 + n].record()
            torch.cuda.synchronize()
        reset = ev[0].elapsed_time(ev[1])
        t = np.array([ev[1 + i].elapsed_time(ev[2 + i]) for i in range(n)]) * 1e3
        tot = ev[0].elapsed_time(ev[1 + n])
        print(f"M={M:3d} window {win}: total {tot:.3f} ms  reset {reset * 1e3:.0f} us  launches {n}  "
              f"mean {t.mean():.1f} us  min {t.min():.1f}  p50 {np.median(t):.1f}  max {t.max():.1f}")
        print("   per-launch us:", " ".join(f"{x:.0f}" for x in t[::4]))


if __name__ == "__main__":
    main()
