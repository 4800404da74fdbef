"""Timeline of the dataflow ensemble launch (FC_TRACE build):
FIRECELL_SO=<trace build> python tools/df_trace.py
Per group: start/end (globaltimer), member, window, CTA, group size."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import _lib as L  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402


def main():
    env = S.make_environment(2048, seed=1)
    dl = F.DeviceLandscape.from_environment(env)
    M = 16
    b = F.FireBatch((2048, 2048), M, max_steps=500)
    b.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, p, 0.3) for p in S.ensemble_ph(M)]))
    b.set_seeds(list(range(M)))
    init = torch.as_tensor(S.center_ignition(2048).astype(np.uint8), device="cuda")
    b.reset(init)
    b.run(dl, 500, window=8)
    b.reset(init)
    trace = torch.zeros(600000 + 4 + 65535 * 4, dtype=torch.int64, device="cuda")
    L.lib().fc_debug_set_trace(trace.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b.run(dl, 500, window=8)
    e1.record()
    torch.cuda.synchronize()
    L.lib().fc_debug_set_trace(None)
    print(f"run {e0.elapsed_time(e1):.3f} ms")
    base = 600000
    n = int(trace[base].item())
    rec = trace[base + 4:base + 4 + 4 * n].view(n, 4).cpu().numpy().astype(np.int64)
    t0 = rec[:, 0].min()
    st, en = (rec[:, 0] - t0) / 1e3, (rec[:, 1] - t0) / 1e3
    m, w = rec[:, 2] >> 20, rec[:, 2] & 0xFFFFF
    print(f"groups {n}, span {en.max():.0f} us, busy CTA-us {np.sum(en - st):.0f} "
          f"(of {296 * en.max():.0f}), mean group {np.mean(en - st):.1f} us")
    for mm in range(0, M, 5):
        sel = m == mm
        ws = np.unique(w[sel])
        ends = np.array([en[sel & (w == x)].max() for x in ws])
        starts = np.array([st[sel & (w == x)].min() for x in ws])
        gaps = starts[1:] - ends[:-1]
        dur = ends - starts
        print(f"member {mm}: windows {len(ws)}, end {ends.max():.0f} us, window dur mean "
              f"{dur.mean():.1f} max {dur.max():.1f}, gap mean {gaps.mean():.2f} max {gaps.max():.2f} us")
    ends_m = [en[m == mm].max() for mm in range(M)]
    print("member end (us):", " ".join(f"{x:.0f}" for x in ends_m))
    crit = int(np.argmax(ends_m))
    sel = m == crit
    ws = np.unique(w[sel])
    rows = []
    for x in ws:
        s2 = sel & (w == x)
        rows.append((x, s2.sum(), st[s2].min(), st[s2].max(), en[s2].min(), en[s2].max(),
                     np.median(en[s2] - st[s2])))
    print(f"critical member {crit}: window, groups, dispatch skew, dur, median group, gap to next")
    for i, (x, ng, s0, s1, e0_, e1_, med) in enumerate(rows):
        gap = rows[i + 1][2] - e1_ if i + 1 < len(rows) else 0.0
        if i % 4 == 0 or i == len(rows) - 1:
            print(f"  w{x:3d} ng {ng:3d} skew {s1 - s0:5.1f} dur {e1_ - s0:5.1f} "
                  f"med {med:5.1f} gap {gap:5.2f}")
    tot_gap = sum(rows[i + 1][2] - rows[i][5] for i in range(len(rows) - 1))
    tot_skew = sum(r[3] - r[2] for r in rows)
    tot_dur = sum(r[5] - r[2] for r in rows)
    print(f"critical member totals: windows {tot_dur:.0f} us, of which dispatch skew {tot_skew:.0f}; "
          f"gaps {tot_gap:.0f} us")
    # concurrency over time
    grid = np.linspace(0, en.max(), 20)
    conc = [int(np.sum((st <= x) & (en > x))) for x in grid]
    print("concurrent groups over time:", conc)


if __name__ == "__main__":
    main()
