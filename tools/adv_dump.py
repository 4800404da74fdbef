"""Dump the device state / J of the adversarial accuracy cases
(tests/test_gpu_envelope.py) for offline analysis against the oracle:
python tools/adv_dump.py OUT.npz"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402
from test_gpu_envelope import ADVERSARIAL, _rough  # noqa: E402

out = {}
for name, (seed, vmax, pr) in sorted(ADVERSARIAL.items()):
    n, steps, members = 160, 80, 2
    env = _rough(n, seed, vmax)
    dl = F.DeviceLandscape.from_environment(env)
    b = F.FireBatch((n, n), members, max_steps=steps, with_jacobian=True)
    b.set_params(F.pack_params(*pr))
    b.set_seeds([seed * 10 + m for m in range(members)])
    b.reset(S.center_ignition(n, block=5))
    b.run(dl, steps, attach=[s % 4 != 3 for s in range(steps)])
    out[name + "_jac"] = b.jac.cpu().numpy()
    out[name + "_acc"] = b.acc.cpu().numpy()
np.savez_compressed(sys.argv[1], **out)
