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
    runner = EnsembleRunner((H, W), M, STEPS, depth=int(os.environ.get("E2E_DEPTH", 2)))
    env_host = torch.stack([torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)) for a in
                            (env.elevation, env.wind_speed, env.wind_direction, env.canopy,
                             env.density)]).pin_memory()
    init_host = torch.from_numpy(S.center_ignition(H).astype(np.uint8)).pin_memory()
    for _ in range(3):
        runner(env_host, init_host, params, list(range(M)))
    torch.cuda.synchronize()
    # timing probes only (wrong results): E2E_PROBE=nolandscape / noexport
    probe = os.environ.get("E2E_PROBE", "")
    if probe == "nolandscape":
        for sl in runner.slots:
            sl.build_landscape = lambda *a: None
    if probe == "noexport":
        for sl in runner.slots:
            sl.export = lambda *a: None
    n = 20
    t0 = time.perf_counter()
    # depth - 1 calls ahead of the host: call i's results are read after
    # call i + depth - 1 is submitted
    pending = []
    for _ in range(n):
        pending.append(runner.submit(env_host, init_host, params, list(range(M))))
        if len(pending) >= len(runner.slots):
            pending.pop(0).result()
    for tk in pending:
        tk.result()
    dt = (time.perf_counter() - t0) / n
    knobs = {k: v for k, v in os.environ.items() if k.startswith(("FC_", "E2E_"))}
    print(f"{knobs or 'default'}: e2e {1e3 * dt:.3f} ms per call, "
          f"{M * H * W * STEPS / dt:.3g} cell-updates/s")


if __name__ == "__main__":
    main()
