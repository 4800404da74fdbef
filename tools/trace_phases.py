"""Per-warp phase timing of the window kernel from an FC_TRACE build:
FIRECELL_SO=<trace build> python tools/trace_phases.py [c1|c3] [launch_index] [warps]

Per (CTA, step, warp): step start, item-phase start (after barrier 1),
item-phase end (before barrier 2), item rounds of the warp."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import _lib as L  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402


def setup(work):
    if work.startswith("c1"):
        env = S.make_environment(2048, seed=1)
        dl = F.DeviceLandscape.from_environment(env)
        M = int(work[3:]) if work.startswith("c1m") else 16  # c1m1: one member
        b = F.FireBatch((2048, 2048), M, max_steps=504)
        ph = S.ensemble_ph(M)
        b.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, p, 0.3) for p in ph]))
        b.set_seeds(list(range(M)))
        b.reset(S.center_ignition(2048))
        return dl, b
    n = 16384
    e = S.make_environment_torch(n, n, seed=3, device="cuda")
    dl = F.DeviceLandscape.from_elevation(e["elevation"], e["wind_speed"], e["wind_direction"],
                                          e["canopy"], e["density"])
    del e
    b = F.FireBatch((n, n), 1, max_steps=504)
    b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.3))
    b.set_seeds([3])
    b.reset(S.random_blocks(n, n, 8, 5, seed=3))
    return dl, b


def main():
    work = sys.argv[1] if len(sys.argv) > 1 else "c1"
    target = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    warps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    dl, b = setup(work)
    trace = torch.zeros((512, 16, warps, 8), dtype=torch.int64, device="cuda")
    for q in range(target + 1):
        if q == target:
            L.lib().fc_debug_set_trace(trace.data_ptr())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        b.run(dl, 8, window=8)
        if q == target:
            e1.record()
            L.lib().fc_debug_set_trace(None)
    torch.cuda.synchronize()
    print(f"{work} launch {target}: {1e3 * e0.elapsed_time(e1):.1f} us")
    tr = trace.cpu().numpy().astype(np.float64)
    cta = tr[:, 15, 0, :4]
    cta = cta[cta[:, 0] > 0]
    if len(cta):
        t0 = cta[:, 0].min()
        ent, ext = (cta[:, 0] - t0) / 1e3, (cta[:, 1] - t0) / 1e3
        print(f"CTAs {len(cta)}, listed tiles {int(cta[0, 3])}: entry spread {ent.max():.1f} us, "
              f"exit p10/p50/p90/max {np.percentile(ext, 10):.1f}/{np.median(ext):.1f}/"
              f"{np.percentile(ext, 90):.1f}/{ext.max():.1f} us, groups per CTA mean "
              f"{cta[:, 2].mean():.2f} max {cta[:, 2].max():.0f}")
    if len(cta) and os.environ.get("TRACE_CORR"):
        # per CTA: chain (entry -> exit), summed per-step item rounds and
        # item-phase critical cycles; which one explains the slowest CTAs?
        full = trace.cpu().numpy().astype(np.float64)
        ok = full[:, 15, 0, 0] > 0
        ch = (full[ok, 15, 0, 1] - full[ok, 15, 0, 0]) / 1e3
        rounds = full[ok, :8, :, 3].max(axis=2).sum(axis=1)
        crit = (full[ok, :8, :, 2].max(axis=2) - full[ok, :8, :, 1].min(axis=2)).clip(0).sum(axis=1)
        swp = (full[ok, :8, :, 1].min(axis=2) - full[ok, :8, :, 0].min(axis=2)).clip(0).sum(axis=1)
        print(f"corr(chain, rounds) {np.corrcoef(ch, rounds)[0, 1]:.2f}  corr(chain, item crit) "
              f"{np.corrcoef(ch, crit)[0, 1]:.2f}  corr(chain, sweep) {np.corrcoef(ch, swp)[0, 1]:.2f}")
        order = np.argsort(ch)
        for lab, idx in (("fastest", order[:5]), ("slowest", order[-5:])):
            for i in idx:
                print(f"  {lab} chain {ch[i]:6.1f} us rounds {rounds[i]:4.0f} item-crit {crit[i]:7.0f} "
                      f"sweep {swp[i]:6.0f} cycles")
    act = tr[:, 0, 0, 0] != 0
    tr = tr[act]
    print("CTAs traced", int(act.sum()))
    # per-CTA chain: first step start -> last recorded item end (first group)
    spans = []
    for c in range(tr.shape[0]):
        st0 = tr[c, 0, :, 0]
        st0 = st0[st0 > 0]
        ends = tr[c, :, :, 2]
        ends = ends[ends > 0]
        if len(st0) and len(ends):
            spans.append(ends.max() - st0.min())
    spans = np.array(spans)
    if len(spans):
        print(f"per-CTA chain cycles: mean {spans.mean():.0f} p50 {np.median(spans):.0f} "
              f"p90 {np.percentile(spans, 90):.0f} max {spans.max():.0f}")
    for s_ in range(8):
        st = tr[:, s_]  # (cta, warp, 4)
        ok = (st[:, :, 1] != 0).all(1) & (st[:, :, 2] != 0).all(1)
        if not ok.any():
            continue
        st = st[ok]
        sweep = st[:, :, 1].min(1) - st[:, :, 0].min(1)        # step start -> barrier-1 release
        items = st[:, :, 2].max(1) - st[:, :, 1].min(1)         # release -> last warp done
        wdur = st[:, :, 2] - st[:, :, 1]
        rounds = st[:, :, 3]
        nxt = (tr[ok][:, s_ + 1, :, 0].min(1) - st[:, :, 2].max(1)) if s_ < 7 else np.zeros(1)
        print(f"step {s_}: CTAs {ok.sum():4d} | start->release {sweep.mean():6.0f} | items crit "
              f"{items.mean():6.0f} (p90 {np.percentile(items, 90):6.0f} max {items.max():6.0f}) | "
              f"warp item dur mean {wdur.mean():6.0f} | rounds mean {rounds.mean():4.2f} max "
              f"{rounds.max():.0f} | tail {nxt.mean():6.0f}")
        it = st.reshape(-1, 8)
        it = it[(it[:, 4] > 0) & (it[:, 7] > 0)]
        if len(it):
            print(f"        candidate item (lane 0): start->entry {np.median(it[:, 4] - it[:, 1]):6.0f} "
                  f"live+draw {np.median(it[:, 5] - it[:, 4]):6.0f} slots {np.median(it[:, 6] - it[:, 5]):6.0f} "
                  f"decide {np.median(it[:, 7] - it[:, 6]):6.0f} (medians over {len(it)} warps)")


if __name__ == "__main__":
    main()
