"""Fixture loading for tests (goldens produced by tests/golden/make_golden.py
from the reference itself)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def meta():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


class P:
    """Minimal params record (c1, c2, a, p_h, p_continue)."""

    def __init__(self, arr):
        self.c1, self.c2, self.a, self.p_h, self.p_continue = (float(v) for v in arr)


RUN_CASES = ["run_rand16", "run_rand9_source", "run_windswap", "run_source_grad",
             "run_radians", "run_partial_attach", "run_windless", "run_ragged",
             "run_saturated"]


def case_kwargs(name, d):
    kw = {}
    if name in ("run_rand9_source", "run_source_grad"):
        kw["factor_site"] = "source"
    if name == "run_radians":
        kw["slope_units"] = "radians"
    if "wind_at" in d:
        kw["wind_schedule"] = [(int(d["wind_at"]), d["wind_speed2"], d["wind_direction2"])]
    return kw
