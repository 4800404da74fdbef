"""Small driver for ncu / compute-sanitizer runs of the step kernels.

    python tools/profile_workloads.py c1 [steps]      # 16 x 2048^2 ensemble, list sweep
    python tools/profile_workloads.py c3dense [steps] # 16384^2 dense sweep
    python tools/profile_workloads.py c3skip [steps]  # 16384^2 activity-list sweep
    python tools/profile_workloads.py c2 [iters]      # calibration iterations
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402


def main():
    mode = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    dev = torch.device("cuda")
    if mode == "c1":
        steps = n or 500
        env = S.make_environment(2048, seed=1)
        dl = F.DeviceLandscape.from_environment(env)
        b = F.FireBatch((2048, 2048), 16, max_steps=steps)
        ph = S.ensemble_ph(16)
        b.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, p, 0.3) for p in ph]))
        b.set_seeds(list(range(16)))
        b.reset(S.center_ignition(2048))
        b.run(dl, steps)
    elif mode in ("c3dense", "c3skip"):
        steps = n or 20
        e = S.make_environment_torch(16384, 16384, seed=3, device=dev)
        dl = F.DeviceLandscape.from_elevation(e["elevation"], e["wind_speed"], e["wind_direction"],
                                              e["canopy"], e["density"])
        b = F.FireBatch((16384, 16384), 1, max_steps=steps)
        b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.3))
        b.set_seeds([3])
        b.reset(S.random_blocks(16384, 16384, 8, 5, seed=3))
        b.run(dl, steps, skip_inactive=(mode == "c3skip"))
    elif mode == "c2":
        iters = n or 3
        env = S.make_environment(1024, seed=2)
        dl = F.DeviceLandscape.from_environment(env)
        b = F.FireBatch((1024, 1024), 1, max_steps=100, with_jacobian=True)
        b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.3))
        b.set_seeds([7])
        tg = torch.zeros((4, 1024, 1024), dtype=torch.uint8, device=dev)
        tg[:, 480:560, 480:560] = 1
        for k in range(1, iters + 1):
            b.reset(S.center_ignition(1024))
            b.run(dl, 100, attach=[True] * 100)
            _, _, g, _ = b.loss_grad(tg, [25, 50, 75, 100])
            b.adamw(g, None, 1e-2)
    torch.cuda.synchronize()
    print("done", mode)


if __name__ == "__main__":
    main()
