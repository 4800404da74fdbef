"""Config-4 iteration breakdown (256 members x 1024^2 x 200 attached steps):
CUDA events around reset, the attached run, the fused loss/gradient and the
AdamW step.  python tools/c4_breakdown.py [members]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402
from paper_2502_18738_b200.device import wind_ramp_schedule  # noqa: E402


def main():
    members = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    n, T = 1024, 200
    env = S.make_environment(n, seed=4)
    dl = F.DeviceLandscape.from_environment(env)
    sched = wind_ramp_schedule(T, 2.0, 12.0, 90.0, device="cuda")
    init = torch.as_tensor(S.center_ignition(n).astype(np.uint8), device="cuda")
    hid = S.HIDDEN_C2_PARAMS
    tb = F.FireBatch((n, n), 1, max_steps=T)
    tb.set_params(F.pack_params(hid["c1"], hid["c2"], hid["a"], hid["p_h"], hid["p_continue"]))
    tb.set_seeds([7])
    tb.reset(init)
    targets = []
    for _ in range(4):
        tb.run(dl, 50, wind_schedule=sched)
        b_, d_ = tb.unpack()
        targets.append(b_[0] | d_[0])
    targets = torch.stack(targets)
    b = F.FireBatch((n, n), members, max_steps=T, with_jacobian=True)
    p0 = S.DEFAULT_BENCH_PARAMS
    b.set_params(F.pack_params(p0["c1"], p0["c2"], p0["a"], p0["p_h"], p0["p_continue"]))
    b.set_seeds(list(range(members)))
    att = [True] * T
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    for rep in range(3):
        ev[0].record()
        b.reset(init)
        ev[1].record()
        b.run(dl, T, attach=att, wind_schedule=sched, window=int(os.environ.get("WINDOW", 8)))
        ev[2].record()
        loss, _, grad, _ = b.loss_grad(targets, [50, 100, 150, 200])
        ev[3].record()
        g = grad.sum(0, keepdim=True)
        ev[4].record()
        torch.cuda.synchronize()
    names = ["reset", "run (attached, wind schedule)", "loss_grad (4 targets)", "grad sum"]
    for i, nm in enumerate(names):
        print(f"{nm:32s} {ev[i].elapsed_time(ev[i + 1]):8.3f} ms")
    cnt = b.counters[:, :T].to(torch.int64).sum((0, 1)).cpu().numpy()
    print("ignitions", cnt[0], "burnouts", cnt[1], "tiles visited", cnt[2], "candidates", cnt[3])


if __name__ == "__main__":
    main()
