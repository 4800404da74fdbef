"""Is the c1 ensemble run latency- or throughput-bound?  Time the c1
workload (2048^2, 500 steps) at M = 1..64 members:
FIRECELL_SO=<so> python tools/scale_members.py"""
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
    for M in [int(x) for x in os.environ.get("MS", "1,4,8,16,32,64").split(",")]:
        b = F.FireBatch((2048, 2048), M, max_steps=500)
        ph = S.ensemble_ph(M)
        b.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, p, 0.3) for p in ph]))
        b.set_seeds(list(range(M)))

        def run():
            b.reset(init)
            b.run(dl, 500, window=8)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"M={M:3d}  {ms:7.3f} ms/run  {ms / M:6.3f} ms/member  "
              f"{M * 2048 * 2048 * 500 / (ms / 1e3):.3e} cu/s")
        del b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
