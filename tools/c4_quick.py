"""Config 4 iteration time (bench.bench_ensemble_calibration) with an
optional window override: WINDOW=4|8 python tools/c4_quick.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_18738_b200 import ensemble  # noqa: E402

w = os.environ.get("WINDOW")
gr = os.environ.get("C4_GRAPH")
if w or gr:
    orig = ensemble.EnsembleCalibrator.__init__

    def init(self, *a, **k):
        if w:
            k["window"] = int(w)
        if gr:
            k["graph"] = bool(int(gr))
        orig(self, *a, **k)
    ensemble.EnsembleCalibrator.__init__ = init
r = bench.bench_ensemble_calibration(torch.device("cuda", 0), 0, 1, iters=5)
print(os.environ.get("FC_DATAFLOW"), "window", w, "graph", gr, "c4 it/s %.1f ms %.3f" % (r["iter_per_s"], r["ms_per_iter"]))
