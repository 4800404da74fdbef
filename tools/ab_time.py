"""Quick A/B timing of builds: FIRECELL_SO=<so> python tools/ab_time.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    window = int(os.environ.get("WINDOW", 8))
    env = S.make_environment(2048, seed=1)
    dl = F.DeviceLandscape.from_environment(env)
    b = F.FireBatch((2048, 2048), 16, max_steps=500)
    ph = S.ensemble_ph(16)
    b.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, p, 0.3) for p in ph]))
    b.set_seeds(list(range(16)))
    init = torch.as_tensor(S.center_ignition(2048).astype(np.uint8), device="cuda")

    def c1():
        b.reset(init)
        b.run(dl, 500, window=window)
    print(os.environ.get("FIRECELL_SO", "default"), "window", window, "c1 ms/run %.3f" % timeit(c1))
    if os.environ.get("AB_GRAPH"):
        g = F.CapturedSequence(c1)
        print("c1 graph replay ms/run %.3f" % timeit(g.replay))
    if os.environ.get("AB_EMPTY"):
        # same launches with no fire anywhere: every CTA finds an empty list
        # and exits, so this is the fixed per-launch cost of the run
        zero = torch.zeros_like(init)

        def c1_empty():
            b.reset(zero)
            b.run(dl, 500, window=window)
        ge = F.CapturedSequence(c1_empty)
        print("c1 no-fire graph replay ms/run %.3f" % timeit(ge.replay))
    n = 1024
    env2 = S.make_environment(n, seed=2)
    dl2 = F.DeviceLandscape.from_environment(env2)
    b2 = F.FireBatch((n, n), 1, max_steps=100, with_jacobian=True)
    b2.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.3))
    b2.set_seeds([7])
    init2 = torch.as_tensor(S.center_ignition(n).astype(np.uint8), device="cuda")

    def c2fwd():
        b2.reset(init2)
        b2.run(dl2, 100, attach=[True] * 100, window=window)
    print("c2 fwd(all attached) ms/iter %.3f" % timeit(c2fwd, 20))
    if os.environ.get("AB_C3"):
        n3 = 16384
        e = S.make_environment_torch(n3, n3, seed=3, device="cuda")
        dl3 = F.DeviceLandscape.from_elevation(e["elevation"], e["wind_speed"], e["wind_direction"],
                                               e["canopy"], e["density"])
        del e
        b3 = F.FireBatch((n3, n3), 1, max_steps=200)
        b3.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.3))
        b3.set_seeds([3])
        init3 = torch.as_tensor(S.random_blocks(n3, n3, 8, 5, seed=3).astype(np.uint8), device="cuda")
        for skip in (True, False):
            def c3():
                b3.reset(init3)
                b3.run(dl3, 200, window=window, skip_inactive=skip)
            print("c3 %s 200 steps ms %.3f" % ("skip" if skip else "dense", timeit(c3, 3)))


if __name__ == "__main__":
    main()
