"""c1 end to end through EnsembleRunner.submit (as bench.py's e2e leg):
pinned host inputs, two calls in flight, results read on the host."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_18738_b200 import synthetic as S  # noqa: E402
from paper_2502_18738_b200.ensemble import EnsembleRunner  # noqa: E402

H = W = 2048
M, STEPS = 16, 500


def main():
    env = S.make_environment(H, seed=1)
    ph = S.ensemble_ph(M)
    params = [(0.045, 0.131, 0.078, float(p), 0.3) for p in ph]
    runner = EnsembleRunner((H, W), M, STEPS)
    env_host = torch.stack([torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)) for a in
                            (env.elevation, env.wind_speed, env.wind_direction, env.canopy,
                             env.density)]).pin_memory()
    init_host = torch.from_numpy(S.center_ignition(H).astype(np.uint8)).pin_memory()
    for _ in range(3):
        runner(env_host, init_host, params, list(range(M)))
    torch.cuda.synchronize()
    n = 20
    t0 = time.perf_counter()
    prev = None
    for _ in range(n):
        tk = runner.submit(env_host, init_host, params, list(range(M)))
        if prev is not None:
            prev.result()
        prev = tk
    prev.result()
    dt = (time.perf_counter() - t0) / n
    print(f"{os.environ.get('FC_DF_CTAS', 'default')}: e2e {1e3 * dt:.3f} ms per call, "
          f"{M * H * W * STEPS / dt:.3g} cell-updates/s")


if __name__ == "__main__":
    main()
