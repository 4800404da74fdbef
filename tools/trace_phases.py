"""Phase timing of the window kernel from an FC_TRACE build:
FIRECELL_SO=<trace build> python tools/trace_phases.py [launch_index]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import _lib as L  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402


def main():
    target = int(sys.argv[1]) if len(sys.argv) > 1 else 55
    env = S.make_environment(2048, seed=1)
    dl = F.DeviceLandscape.from_environment(env)
    b = F.FireBatch((2048, 2048), 16, max_steps=504)
    ph = S.ensemble_ph(16)
    b.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, p, 0.3) for p in ph]))
    b.set_seeds(list(range(16)))
    b.reset(S.center_ignition(2048))
    trace = torch.zeros((512, 16, 4), dtype=torch.int64, device="cuda")
    for q in range(63):
        if q == target:
            L.lib().fc_debug_set_trace(trace.data_ptr())
        b.run(dl, 8, window=8)
        if q == target:
            L.lib().fc_debug_set_trace(None)
    torch.cuda.synchronize()
    tr = trace.cpu().numpy()
    act = tr[:, 0, 0] != 0
    tr = tr[act]
    print("CTAs traced", act.sum())
    bit = tr[:, :, 1] - tr[:, :, 0]
    item = tr[:, :, 2] - tr[:, :, 1]
    nxt = tr[:, 1:, 0] - tr[:, :-1, 2]
    valid = (tr[:, :, 0] != 0) & (tr[:, :, 2] != 0)
    for s_ in range(8):
        v = valid[:, s_]
        if not v.any():
            continue
        print(f"step {s_}: bit phase mean {bit[v, s_].mean():8.0f} max {bit[v, s_].max():8.0f} cyc | "
              f"items mean {item[v, s_].mean():8.0f} max {item[v, s_].max():8.0f} cyc | "
              f"pool mean {tr[v, s_, 3].mean():6.0f} max {tr[v, s_, 3].max():6.0f}")
    print("tail (update) mean", nxt[valid[:, 1:]].mean() if valid[:, 1:].any() else None)
    ok = (tr[:, :, 0] != 0).all(1) & (tr[:, :, 2] != 0).all(1)
    span = tr[ok][:, :, 2].max(1) - tr[ok][:, 0, 0]
    print("per-CTA span (first group) mean", span.mean(), "max", span.max(), "p90", np.percentile(span, 90))
    print("step-time per CTA (bit+items+tail) mean", (tr[ok][:, 1:, 0] - tr[ok][:, :-1, 0]).mean())


if __name__ == "__main__":
    main()
