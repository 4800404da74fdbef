"""Config-2 calibration iteration (bench.py's bench_calibration) replayed a
few times as one CUDA graph, for a launch list:
ncu --metrics gpu__time_duration.sum --csv python tools/c2_launches.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    r = bench.bench_calibration("cuda")
    print({k: r[k] for k in ("iter_per_s", "ms_per_iter")})
