"""c1 e2e pipeline timeline (as tools/e2e_quick.py): CUDA events around each
call's upload + landscape build (upload stream), reset + run (compute
stream) and export (copy stream), reported relative to the run's start."""
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


def ev(stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


def main():
    env = S.make_environment(H, seed=1)
    ph = S.ensemble_ph(M)
    params = [(0.045, 0.131, 0.078, float(p), 0.3) for p in ph]
    runner = EnsembleRunner((H, W), M, STEPS, depth=int(os.environ.get("E2E_DEPTH", 2)))
    env_host = torch.stack([torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)) for a in
                            (env.elevation, env.wind_speed, env.wind_direction, env.canopy,
                             env.density)]).pin_memory()
    init_host = torch.from_numpy(S.center_ignition(H).astype(np.uint8)).pin_memory()
    for _ in range(max(3, len(runner.slots))):
        runner(env_host, init_host, params, list(range(M)))
    torch.cuda.synchronize()
    marks = []
    for sl in runner.slots:
        bl, ex, dp = sl.build_landscape, sl.export, sl.graph.replay

        def build(stream, ctas, _bl=bl):
            marks.append(("land0", ev(stream)))
            _bl(stream, ctas)
            marks.append(("land1", ev(stream)))

        def export(stream, _ex=ex):
            marks.append(("exp0", ev(stream)))
            _ex(stream)
            marks.append(("exp1", ev(stream)))

        def replay(_dp=dp):
            s = torch.cuda.current_stream()
            marks.append(("run0", ev(s)))
            _dp()
            marks.append(("run1", ev(s)))
        sl.build_landscape, sl.export, sl.graph.replay = build, export, replay
    n = 12
    t0 = time.perf_counter()
    pending = []
    for _ in range(n):
        pending.append(runner.submit(env_host, init_host, params, list(range(M))))
        if len(pending) >= len(runner.slots):
            pending.pop(0).result()
    for tk in pending:
        tk.result()
    dt = (time.perf_counter() - t0) / n
    torch.cuda.synchronize()
    ref = next(e for k, e in marks if k == "run0")
    rows = [(k, ref.elapsed_time(e)) for k, e in marks]
    rows.sort(key=lambda r: r[1])
    if os.environ.get("E2E_VERBOSE"):
        for k, t in rows:
            print(f"{t:9.3f} ms  {k}")
    r0 = sorted(t for k, t in rows if k == "run0")
    r1 = sorted(t for k, t in rows if k == "run1")
    gaps = [a - b for a, b in zip(r0[1:], r1)]
    print("gaps run end -> next run start (ms):", " ".join(f"{g:.3f}" for g in gaps))
    d = {}
    for k, t in [(k, ref.elapsed_time(e)) for k, e in marks]:
        d.setdefault(k, []).append(t)
    for a in ("land", "run", "exp"):
        x = np.array(d[a + "1"][: len(d[a + "0"])]) - np.array(d[a + "0"][: len(d[a + "1"])])
        print(f"{a}: mean {x.mean():.3f} ms  min {x.min():.3f}  max {x.max():.3f}")
    print(f"e2e {1e3 * dt:.3f} ms per call")


if __name__ == "__main__":
    main()
