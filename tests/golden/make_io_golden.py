"""Generate tests/golden/io/ by running the REFERENCE's data_io and CLI.

Run here (the build container, where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_io_golden.py

Everything under tests/golden/io/ is written by pyrocell 0.1.0 itself
(/root/reference/pkg/src): PTFG grids of each dtype and rank
(data_io.write_grid), two landscape bundles (data_io.write_landscape), the
output directories of ``pyrocell simulate`` / ``calibrate`` and the stdout
of ``pyrocell metrics``, plus io.json with sha256 fingerprints of the fp64
synthetic landscapes (synthetic.make_landscape) and of slope_from_altitude
/ wind_from_uv / pad_nonburnable / render_state outputs.  Nothing at test
time reads /root/reference.
"""
from __future__ import annotations

import contextlib
import hashlib
import io
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
sys.path.insert(0, "/root/reference/pkg/src")

from pyrocell import cli, data_io, synthetic  # noqa: E402  (the reference)
from pyrocell.model import FireState  # noqa: E402


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(str(a.dtype).encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def run_cli(*argv) -> str:
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = cli.main([str(a) for a in argv])
    assert code == 0, argv
    return buf.getvalue()


def main():
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    rng = np.random.default_rng(20250218)
    meta = {"grids": {}, "landscapes": {}, "helpers": {}}

    # ---- PTFG grids
    grids = {
        "f32_2d": rng.standard_normal((7, 5)).astype(np.float32),
        "f64_2d": rng.uniform(-1e3, 1e3, (4, 9)),            # stored as float32
        "bool_2d": rng.uniform(size=(6, 11)) < 0.4,
        "f32_1d": rng.standard_normal(13).astype(np.float32),
        "f32_3d": rng.standard_normal((3, 4, 2)).astype(np.float32),
        "f32_4d": rng.standard_normal((2, 3, 3, 3)).astype(np.float32),
        "int_2d": rng.integers(-50, 50, (3, 3)),             # stored as float32
        "bool_empty": np.zeros((0, 4), dtype=bool),
    }
    for name, g in grids.items():
        data_io.write_grid(g, os.path.join(OUT, f"{name}.ptfg"))
        np.save(os.path.join(OUT, f"{name}.npy"), g)
    # ---- landscape bundles
    data_io.write_landscape(synthetic.make_landscape("hill", 24), os.path.join(OUT, "bundle_hill"))
    data_io.write_landscape(
        synthetic.make_landscape("random:5", 20, slope_sign="uphill-positive"),
        os.path.join(OUT, "bundle_random"))
    # ---- fingerprints of the synthetic generators (fp64, size 17)
    for kind in ("flat", "hill", "valley", "windy", "random:3"):
        for sign in ("downhill-positive", "uphill-positive"):
            land = synthetic.make_landscape(kind, 17, slope_sign=sign)
            meta["landscapes"][f"{kind}|{sign}"] = {
                f: sha(getattr(land, f)) for f in
                ("wind_speed", "wind_direction", "slope", "canopy", "density")}
    alt = rng.uniform(0, 400, (9, 12))
    meta["helpers"]["slope_from_altitude"] = sha(data_io.slope_from_altitude(alt, 25.0))
    meta["helpers"]["slope_from_altitude_uphill"] = sha(
        data_io.slope_from_altitude(alt, 25.0, "uphill-positive"))
    np.save(os.path.join(OUT, "altitude.npy"), alt)
    u, v = rng.standard_normal((2, 6, 7)) * 5
    np.save(os.path.join(OUT, "uv.npy"), np.stack([u, v]))
    s, d = data_io.wind_from_uv(u, v)
    meta["helpers"]["wind_from_uv"] = [sha(s), sha(d)]
    pad = data_io.pad_nonburnable(synthetic.make_landscape("hill", 9), 2)
    meta["helpers"]["pad_nonburnable"] = {
        f: sha(getattr(pad, f)) for f in
        ("wind_speed", "wind_direction", "slope", "canopy", "density")}
    land = synthetic.make_landscape("random:4", 12)
    st = FireState(rng.uniform(size=(12, 12)) < 0.2, rng.uniform(size=(12, 12)) < 0.2,
                   np.zeros((12, 12)), 0)
    st.burned &= ~st.burning
    np.save(os.path.join(OUT, "render_masks.npy"), np.stack([st.burning, st.burned]))
    meta["helpers"]["render_state"] = sha(data_io.render_state(st, land))

    # ---- CLI runs
    sim1 = os.path.join(OUT, "sim_windy")
    run_cli("simulate", "--synthetic", "windy", "--size", 32, "--steps", 12, "--seed", 3,
            "--snapshot-every", 6, "--threads", 1, "--out", sim1)
    sim2 = os.path.join(OUT, "sim_bundle")
    run_cli("simulate", "--landscape", os.path.join(OUT, "bundle_random"), "--steps", 10,
            "--seed", 2, "--p-h", 0.7, "--factor-site", "source", "--threads", 1, "--out", sim2)
    sim3 = os.path.join(OUT, "sim_zero")
    run_cli("simulate", "--synthetic", "flat", "--size", 16, "--steps", 0, "--seed", 1,
            "--threads", 1, "--out", sim3)
    meta["metrics_stdout"] = run_cli(
        "metrics", "--pred", os.path.join(sim1, "affected_00006.ptfg"),
        "--pred", os.path.join(sim1, "affected_00012.ptfg"),
        "--target", os.path.join(sim1, "affected_00012.ptfg"),
        "--target", os.path.join(sim1, "final_burning.ptfg"))
    cal = os.path.join(OUT, "cal_windy")
    run_cli("calibrate", "--synthetic", "windy", "--size", 32, "--p-h", 0.3,
            "--max-epochs", 2, "--lr", 0.02, "--seed", 5, "--steps-update-interval", 6,
            "--target", os.path.join(sim1, "affected_00006.ptfg"),
            "--target", os.path.join(sim1, "affected_00012.ptfg"),
            "--threads", 1, "--out", cal)
    meta["cli_argv"] = {
        "sim_windy": "simulate --synthetic windy --size 32 --steps 12 --seed 3 "
                     "--snapshot-every 6 --threads 1",
        "sim_bundle": "simulate --landscape bundle_random --steps 10 --seed 2 --p-h 0.7 "
                      "--factor-site source --threads 1",
        "sim_zero": "simulate --synthetic flat --size 16 --steps 0 --seed 1 --threads 1",
        "cal_windy": "calibrate --synthetic windy --size 32 --p-h 0.3 --max-epochs 2 --lr 0.02 "
                     "--seed 5 --steps-update-interval 6 --target sim_windy/affected_00006.ptfg "
                     "--target sim_windy/affected_00012.ptfg --threads 1",
    }
    with open(os.path.join(OUT, "io.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
