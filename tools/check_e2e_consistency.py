"""The c1 workload three ways -- FireBatch on device inputs, EnsembleRunner
synchronous calls, EnsembleRunner pipelined submits -- must give identical
final states, accumulators and series.  python tools/check_e2e_consistency.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402
from paper_2502_18738_b200.ensemble import EnsembleRunner  # noqa: E402


def main():
    H, M, STEPS = 2048, 16, 500
    env = S.make_environment(H, seed=1)
    ph = S.ensemble_ph(M)
    params = [(0.045, 0.131, 0.078, float(p), 0.3) for p in ph]
    members = list(range(M))
    init = S.center_ignition(H)
    b = F.FireBatch((H, H), M, max_steps=STEPS)
    b.set_params(np.array([F.pack_params(*p) for p in params]))
    b.set_seeds(members)
    dl = F.DeviceLandscape.from_environment(env)
    ref = []
    for rep in range(2):
        b.reset(init)
        b.run(dl, STEPS, window=8)
        bu, bd = b.unpack()
        ref.append((bu.cpu().numpy(), bd.cpu().numpy(), b.acc.cpu().numpy(), b.series()))
        print("FireBatch rep", rep, "member0 final burning", ref[-1][3][0, -1, 0],
              "affected", int((ref[-1][0] | ref[-1][1]).sum()))
    for x, y in zip(ref[0], ref[1]):
        assert np.array_equal(x, y), "FireBatch not deterministic"
    env_host = torch.stack([torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)) for a in
                            (env.elevation, env.wind_speed, env.wind_direction, env.canopy,
                             env.density)]).pin_memory()
    init_host = torch.from_numpy(init.astype(np.uint8)).pin_memory()
    r = EnsembleRunner((H, H), M, STEPS)
    outs = []
    for k in range(3):
        o = r(env_host, init_host, params, members)
        outs.append(("sync", k, [a.copy() for a in (o.burning, o.burned, o.accumulator, o.series)]))
    tickets = [r.submit(env_host, init_host, params, members)]
    for k in range(5):
        tickets.append(r.submit(env_host, init_host, params, members))
        o = tickets[-2].result()
        outs.append(("pipe", k, [a.copy() for a in (o.burning, o.burned, o.accumulator, o.series)]))
    bad = 0
    for kind, k, arrs in outs:
        same = [np.array_equal(x, y) for x, y in zip(arrs, ref[0])]
        print(kind, k, "member0 final burning", arrs[3][0, -1, 0], "equal", same)
        bad += not all(same)
    print("MISMATCHES", bad)


if __name__ == "__main__":
    main()
