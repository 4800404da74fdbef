"""The stencil in its dense regime: config 3's 16384^2 landscape with fire
everywhere -- a random half of the cells burning at step 0 and burning on
(p_continue 0.999), ignition rare (p_h 0.2) -- so every 32x32 tile is listed
and every cell is a burning cell (continue draw) or a candidate with its
live slots evaluated, in every step, launch after launch.  K = 8 fused steps per launch, activity lists (all tiles
live).  Prints per-launch device time and cell-updates/s; run under ncu for
DRAM bytes.  python tools/dense_regime.py [launches]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402


def main():
    launches = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    # SWEEP=dense: every launch rescans the domain (skip_inactive=False), the
    # mode whose kernels take dense tiles' continue draws in the sweep
    skip = os.environ.get("SWEEP", "list") != "dense"
    n, K = 16384, int(os.environ.get("K", 8))
    e = S.make_environment_torch(n, n, seed=3)
    dl = F.DeviceLandscape.from_elevation(e["elevation"], e["wind_speed"], e["wind_direction"],
                                          e["canopy"], e["density"])
    del e
    gen = torch.Generator(device="cuda")
    gen.manual_seed(11)
    init = (torch.rand((n, n), generator=gen, device="cuda") < 0.5).to(torch.uint8)
    b = F.FireBatch((n, n), 1, max_steps=K * (launches + 2))
    b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.2, 0.999))
    b.set_seeds([3])
    b.reset(init)
    b.run(dl, K, window=K, skip_inactive=skip)  # warm-up launch
    torch.cuda.synchronize()
    evs = []
    for _ in range(launches):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.run(dl, K, window=K, skip_inactive=skip)
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(c) for a, c in evs])
    cnt = b.counters[0, :b.t].to(torch.int64).cpu().numpy()
    tiles = cnt[K::K, 2]
    cu = n * n * K
    print(f"per launch {ms.mean():.3f} ms (min {ms.min():.3f}), tiles visited {tiles.mean():.0f} of "
          f"{(n // 32) ** 2}, {cu / (ms.mean() / 1e3):.3g} cell-updates/s, "
          f"{int(cnt[-1, 0])} ignitions and {int(cnt[-1, 3])} candidates in the last step")


if __name__ == "__main__":
    main()
