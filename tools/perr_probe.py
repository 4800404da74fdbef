"""Worst fp32-vs-fp64 error of the ignition probability over every decision
of several workloads (FC_DEBUG_PERR build):
FIRECELL_SO=<probe build> python tools/perr_probe.py"""
import os
import struct
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import _lib as L  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402
from paper_2502_18738_b200.device import wind_ramp_schedule  # noqa: E402


def f32(bits):
    return struct.unpack("<f", struct.pack("<I", int(bits) & 0xFFFFFFFF))[0]


def probe(name, dl, shape, members, steps, params, wind=None, attach=False):
    buf = torch.zeros(32, dtype=torch.int64, device="cuda")
    b = F.FireBatch(shape, members, max_steps=steps, with_jacobian=attach)
    b.set_params(np.array([F.pack_params(*p) for p in params]))
    b.set_seeds(list(range(members)))
    b.reset(S.center_ignition(*shape))
    L.lib().fc_debug_set_trace(buf.data_ptr())
    b.run(dl, steps, wind_schedule=wind, attach=[attach] * steps if attach else None)
    torch.cuda.synchronize()
    L.lib().fc_debug_set_trace(None)
    v = buf.cpu().numpy()
    print(f"{name:40s} decisions {v[1]:>11d}  max |p32-p64| {f32(v[0]):.3e}  max rel {f32(v[2]):.3e}"
          f"  wide recomputes {v[3]}")
    # max relative error (p >= FC_GUARD) per slot-magnitude octave eb in [2^(b-3), 2^(b-2))
    print("    " + "  ".join(f"E<{2.0 ** (b - 2):g}:{f32(v[8 + b]):.1e}" for b in range(24) if v[8 + b]))


def main():
    env = S.make_environment(1024, seed=1)
    dl = F.DeviceLandscape.from_environment(env)
    ph = S.ensemble_ph(8)
    probe("c1-like 8 x 1024^2 x 300", dl, (1024, 1024), 8, 300,
          [(0.045, 0.131, 0.078, p, 0.3) for p in ph])
    sched = wind_ramp_schedule(200, 2.0, 12.0, 90.0, device="cuda")
    probe("c4-like wind ramp 2->12, attached", dl, (1024, 1024), 8, 200,
          [(0.045, 0.131, 0.078, 0.58, 0.3)] * 8, wind=sched, attach=True)
    # extreme parameters: strong slope and wind sensitivity, saturating p_h
    probe("extreme a=1 c1=1 c2=1 p_h=1", dl, (1024, 1024), 4, 200,
          [(1.0, 1.0, 1.0, 1.0, 0.5)] * 4)
    probe("weak a=0.01 c1=0.01 c2=0.01 p_h=0.2", dl, (1024, 1024), 4, 300,
          [(0.01, 0.01, 0.01, 0.2, 0.9)] * 4)
    rng = np.random.default_rng(3)
    n = 512
    steep = S.make_environment(n, seed=9)
    elev = (rng.random((n, n)) * 3000).astype(np.float32)  # white-noise terrain: slopes near +-89 deg
    spd = (rng.random((n, n)) * 30).astype(np.float32)
    dl2 = F.DeviceLandscape.from_elevation(elev, spd, steep.wind_direction, steep.canopy, steep.density)
    probe("rough terrain, 0-30 m/s wind", dl2, (n, n), 4, 200,
          [(0.045, 0.131, 0.078, 0.58, 0.3), (0.2, 0.3, 0.3, 0.9, 0.3),
           (0.0, 0.0, 0.0, 0.3, 0.3), (1.0, 1.0, 1.0, 1.0, 0.3)])
    probe("rough terrain, attached", dl2, (n, n), 4, 200,
          [(0.045, 0.131, 0.078, 0.58, 0.3), (0.2, 0.3, 0.3, 0.9, 0.3),
           (0.0, 0.0, 0.0, 0.3, 0.3), (1.0, 1.0, 1.0, 1.0, 0.3)], attach=True)
    for c in (0.05, 0.1, 0.2, 0.5):
        probe(f"rough terrain, a=c1=c2={c}", dl2, (n, n), 4, 200, [(c, c, c, 0.6, 0.4)] * 4)


if __name__ == "__main__":
    main()
