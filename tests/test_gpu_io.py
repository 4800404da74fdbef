"""Device-side grid/bundle I/O and the GPU CLI against files the reference
wrote (tests/golden/io, tests/golden/make_io_golden.py).  Bar: grids, series,
snapshots and manifests byte-identical to the reference CLI's; the fp32
accumulator file within RTOL_ACC of the reference's fp64 accumulator
rounded to fp32 (north_star tolerance); calibration numbers within the
tolerances of test_gpu_parity.test_calibrate_golden."""
import os
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2502_18738_b200 as F
from paper_2502_18738_b200 import cli, data_io
from paper_2502_18738_b200.device import DeviceLandscape, FireBatch, pack_params
from paper_2502_18738_b200.synthetic import center_ignition, make_landscape

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "io"
RTOL_ACC = 1e-5
GRIDS = ("f32_2d", "f64_2d", "bool_2d", "f32_1d", "f32_3d", "f32_4d", "int_2d", "bool_empty")


@pytest.mark.parametrize("name", GRIDS)
def test_read_grid_device_equals_host(name):
    host = data_io.read_grid(GOLD / f"{name}.ptfg")
    dev = data_io.read_grid_device(GOLD / f"{name}.ptfg")
    assert dev.is_cuda and tuple(dev.shape) == host.shape
    if host.dtype == bool:
        assert dev.dtype == torch.uint8
        assert np.array_equal(dev.cpu().numpy(), host.astype(np.uint8))
    else:
        assert dev.dtype == torch.float32
        assert dev.cpu().numpy().tobytes() == host.tobytes()


@pytest.mark.parametrize("name", GRIDS)
def test_write_grid_device_bytes(tmp_path, name):
    src = np.load(GOLD / f"{name}.npy")
    t = torch.as_tensor(src).cuda()
    data_io.write_grid_device(t, tmp_path / "g.ptfg")
    assert (tmp_path / "g.ptfg").read_bytes() == (GOLD / f"{name}.ptfg").read_bytes()


def test_read_bool_grid_nonzero_bytes(tmp_path):
    blob = bytearray((GOLD / "bool_2d.ptfg").read_bytes())
    blob[-1] = 7                       # any non-zero byte reads as burning
    (tmp_path / "b.ptfg").write_bytes(bytes(blob))
    dev = data_io.read_grid_device(tmp_path / "b.ptfg")
    assert int(dev.view(-1)[-1]) == 1
    assert np.array_equal(dev.cpu().numpy().astype(bool), data_io.read_grid(tmp_path / "b.ptfg"))


def _states(land, init, steps, seed, params):
    b = FireBatch(land.shape, 1, max_steps=steps)
    b.set_params(pack_params(*params))
    b.set_seeds([seed])
    b.reset(init)
    b.run(land, steps)
    bu, bd = b.unpack()
    return bu.clone(), bd.clone(), b.acc.clone(), b.series()


@pytest.mark.parametrize("bundle", ["bundle_hill", "bundle_random"])
@pytest.mark.parametrize("site", ["target", "source"])
def test_bundle_device_landscape_equals_host_path(bundle, site):
    """read_landscape_device == from_slope_tensor(read_landscape): same
    kernel-layout tensors bit for bit, same runs."""
    a = data_io.read_landscape_device(GOLD / bundle, factor_site=site)
    host = data_io.read_landscape(GOLD / bundle)
    b = DeviceLandscape.from_slope_tensor(host.wind_speed, host.wind_direction, host.slope,
                                          host.canopy, host.density, cell_side=host.cell_side,
                                          factor_site=site)
    for name in ("env", "env64", "slope32", "slope64", "dir32"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    init = center_ignition(*host.shape)
    p = (0.045, 0.131, 0.078, 0.9, 0.5)
    ra, rb = _states(a, init, 15, 4, p), _states(b, init, 15, 4, p)
    for x, y in zip(ra, rb):
        assert np.array_equal(np.asarray(x.cpu() if torch.is_tensor(x) else x),
                              np.asarray(y.cpu() if torch.is_tensor(y) else y))


def test_bundle_radians(tmp_path):
    land = make_landscape("hill", 12)
    rad = F.Landscape(land.wind_speed, land.wind_direction, np.radians(land.slope),
                      land.canopy, land.density, land.cell_side)
    data_io.write_landscape(rad, tmp_path)
    a = data_io.read_landscape_device(tmp_path, slope_units="radians")
    back = data_io.read_landscape(tmp_path)
    b = DeviceLandscape.from_slope_tensor(back.wind_speed, back.wind_direction, back.slope,
                                          back.canopy, back.density, slope_units="radians")
    assert torch.equal(a.slope64, b.slope64)


def _compare_dirs(got: Path, want: Path, skip_manifest_keys=()):
    names = sorted(p.name for p in want.iterdir())
    assert sorted(p.name for p in got.iterdir()) == names
    for n in names:
        if n == "accumulator.ptfg":
            ga, wa = data_io.read_grid(got / n), data_io.read_grid(want / n)
            assert np.array_equal(ga != 0, wa != 0)
            np.testing.assert_allclose(ga, wa, rtol=RTOL_ACC, atol=0)
        elif n == "manifest.txt":
            gm, wm = data_io.read_manifest(got / n), data_io.read_manifest(want / n)
            for k in skip_manifest_keys:
                gm.pop(k, None), wm.pop(k, None)
            assert gm == wm
        else:
            assert (got / n).read_bytes() == (want / n).read_bytes(), n


def test_cli_simulate_windy_matches_reference(tmp_path, capsys):
    out = tmp_path / "sim"
    assert cli.main(["simulate", "--synthetic", "windy", "--size", "32", "--steps", "12",
                     "--seed", "3", "--snapshot-every", "6", "--threads", "1",
                     "--out", str(out)]) == 0
    _compare_dirs(out, GOLD / "sim_windy")
    series = (out / "series.csv").read_text().splitlines()
    assert capsys.readouterr().out.strip().endswith(series[-1].split(",")[3])


def test_cli_simulate_bundle_matches_reference(tmp_path):
    out = tmp_path / "sim"
    assert cli.main(["simulate", "--landscape", str(GOLD / "bundle_random"), "--steps", "10",
                     "--seed", "2", "--p-h", "0.7", "--factor-site", "source", "--threads", "1",
                     "--out", str(out)]) == 0
    _compare_dirs(out, GOLD / "sim_bundle", skip_manifest_keys=("landscape",))


def test_cli_simulate_zero_steps(tmp_path):
    out = tmp_path / "sim"
    assert cli.main(["simulate", "--synthetic", "flat", "--size", "16", "--steps", "0",
                     "--seed", "1", "--threads", "1", "--out", str(out)]) == 0
    _compare_dirs(out, GOLD / "sim_zero")


def test_cli_simulate_deterministic_and_config(tmp_path):
    cfg = tmp_path / "run.cfg"
    cfg.write_text("synthetic=random:2\nsize=40\nsteps=9\nseed=5\np_h=0.8\n")
    outs = []
    for name, extra in (("a", []), ("b", ["--steps", "9"])):
        out = tmp_path / name
        assert cli.main(["simulate", "--config", str(cfg), "--out", str(out)] + extra) == 0
        outs.append({p.name: p.read_bytes() for p in sorted(out.iterdir())})
    assert outs[0] == outs[1]
    m = data_io.read_manifest(tmp_path / "a" / "manifest.txt")
    assert (m["steps"], m["seed"], m["p_h"]) == ("9", "5", "0.8")


def test_cli_calibrate_matches_reference(tmp_path):
    out = tmp_path / "cal"
    sim = GOLD / "sim_windy"
    assert cli.main(["calibrate", "--synthetic", "windy", "--size", "32", "--p-h", "0.3",
                     "--max-epochs", "2", "--lr", "0.02", "--seed", "5",
                     "--steps-update-interval", "6",
                     "--target", str(sim / "affected_00006.ptfg"),
                     "--target", str(sim / "affected_00012.ptfg"),
                     "--threads", "1", "--out", str(out)]) == 0
    want = GOLD / "cal_windy"

    def table(p):
        lines = p.read_text().splitlines()
        return lines[0], np.array([[float(x) for x in ln.split(",")] for ln in lines[1:]])

    for name, rtol in (("metrics.csv", 1e-5), ("trajectory.csv", 1e-4)):
        gh, g = table(out / name)
        wh, w = table(want / name)
        assert gh == wh and g.shape == w.shape
        np.testing.assert_array_equal(g[:, :2], w[:, :2])
        np.testing.assert_allclose(g[:, 2:], w[:, 2:], rtol=rtol, atol=1e-6)
    gb, wb = (data_io.read_manifest(d / "best_params.txt") for d in (out, want))
    assert gb.keys() == wb.keys()
    for k in gb:
        assert float(gb[k]) == pytest.approx(float(wb[k]), rel=1e-4, abs=1e-6)
    gm, wm = (data_io.read_manifest(d / "manifest.txt") for d in (out, want))
    assert float(gm.pop("best_loss")) == pytest.approx(float(wm.pop("best_loss")), rel=1e-5)
    assert gm == wm


def test_cli_bench_rows(tmp_path):
    out = tmp_path / "bench.csv"
    assert cli.main(["bench", "--sizes", "64", "--steps", "20", "--out", str(out)]) == 0
    assert out.read_text().splitlines()[0] == "size,threads,seconds"  # the reference's format
    assert cli.main(["bench", "--sizes", "64,200", "--steps", "30", "--threads", "1,2",
                     "--out", str(out), "--device-times"]) == 0
    rows = out.read_text().splitlines()
    assert rows[0] == "size,threads,seconds,device_seconds"
    assert [r.split(",")[:2] for r in rows[1:]] == [["64", "1"], ["64", "2"], ["200", "1"],
                                                    ["200", "2"]]
    assert all(float(r.split(",")[2]) > 0 and float(r.split(",")[3]) > 0 for r in rows[1:])
