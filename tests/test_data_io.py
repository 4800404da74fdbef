"""data_io / synthetic / CLI host logic against fixtures the reference wrote
(tests/golden/io, made by tests/golden/make_io_golden.py from pyrocell
0.1.0's data_io.write_grid, write_landscape and its CLI).  The reference's
own test list for this module is tests/test_data_io.py:36-301; the cases
below cover the same behaviours.  No GPU needed."""
import hashlib
import json
import os
import struct

import numpy as np
import pytest

from paper_2502_18738_b200 import cli, data_io, synthetic
from paper_2502_18738_b200.kernel import StepStats
from paper_2502_18738_b200.model import FireState, Landscape

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
META = json.load(open(os.path.join(GOLD, "io.json")))
GRIDS = ("f32_2d", "f64_2d", "bool_2d", "f32_1d", "f32_3d", "f32_4d", "int_2d", "bool_empty")
FIELDS = ("wind_speed", "wind_direction", "slope", "canopy", "density")


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(str(a.dtype).encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def gold(*p):
    return os.path.join(GOLD, *p)


# ---------------------------------------------------------------- PTFG grids
@pytest.mark.parametrize("name", GRIDS)
def test_reads_reference_files(name):
    src = np.load(gold(f"{name}.npy"))
    got = data_io.read_grid(gold(f"{name}.ptfg"))
    if src.dtype == bool:
        assert got.dtype == bool and np.array_equal(got, src)
    else:
        assert got.dtype == np.float32
        assert np.array_equal(got, src.astype(np.float32))


@pytest.mark.parametrize("name", GRIDS)
def test_writes_reference_bytes(tmp_path, name):
    data_io.write_grid(np.load(gold(f"{name}.npy")), tmp_path / "g.ptfg")
    assert (tmp_path / "g.ptfg").read_bytes() == open(gold(f"{name}.ptfg"), "rb").read()


def test_float_round_trip_bit_exact(tmp_path):
    g = np.array([[0.0, -0.0, np.inf], [np.nan, 1e-45, 3.4e38]], dtype=np.float32)
    data_io.write_grid(g, tmp_path / "f.ptfg")
    back = data_io.read_grid(tmp_path / "f.ptfg")
    assert back.tobytes() == g.tobytes()


def test_header_layout(tmp_path):
    data_io.write_grid(np.zeros((3, 5), dtype=bool), tmp_path / "h.ptfg")
    blob = (tmp_path / "h.ptfg").read_bytes()
    assert blob[:4] == b"PTFG"
    assert struct.unpack("<HBB", blob[4:8]) == (1, 1, 2)
    assert struct.unpack("<2I", blob[8:16]) == (3, 5)
    assert len(blob) == 16 + 15


def test_bad_magic(tmp_path):
    (tmp_path / "x.ptfg").write_bytes(b"NOPE" + bytes(12))
    with pytest.raises(data_io.BadMagicError, match="not a PTFG grid file"):
        data_io.read_grid(tmp_path / "x.ptfg")
    (tmp_path / "y.ptfg").write_bytes(b"PTF")
    with pytest.raises(data_io.BadMagicError):
        data_io.read_grid(tmp_path / "y.ptfg")


def test_truncated_payload(tmp_path):
    blob = open(gold("f32_2d.ptfg"), "rb").read()
    (tmp_path / "t.ptfg").write_bytes(blob[:-3])
    with pytest.raises(data_io.TruncatedPayloadError, match="expected 140"):
        data_io.read_grid(tmp_path / "t.ptfg")
    (tmp_path / "h.ptfg").write_bytes(blob[:10])
    with pytest.raises(data_io.TruncatedPayloadError, match="truncated header"):
        data_io.read_grid(tmp_path / "h.ptfg")
    (tmp_path / "long.ptfg").write_bytes(blob + b"\0")
    with pytest.raises(data_io.TruncatedPayloadError):
        data_io.read_grid(tmp_path / "long.ptfg")


def test_unknown_dtype_code_and_version(tmp_path):
    blob = bytearray(open(gold("bool_2d.ptfg"), "rb").read())
    blob[6] = 7
    (tmp_path / "d.ptfg").write_bytes(bytes(blob))
    with pytest.raises(data_io.UnsupportedDtypeError, match="unknown dtype code 7"):
        data_io.read_grid(tmp_path / "d.ptfg")
    blob = bytearray(open(gold("bool_2d.ptfg"), "rb").read())
    blob[4] = 2
    (tmp_path / "v.ptfg").write_bytes(bytes(blob))
    with pytest.raises(data_io.GridFileError, match="unsupported version 2"):
        data_io.read_grid(tmp_path / "v.ptfg")


def test_write_rejects_rank0_and_strings(tmp_path):
    with pytest.raises(data_io.GridFileError):
        data_io.write_grid(np.float32(1.0), tmp_path / "s.ptfg")
    with pytest.raises(data_io.UnsupportedDtypeError):
        data_io.write_grid(np.array(["a", "b"]), tmp_path / "s.ptfg")
    assert issubclass(data_io.GridFileError, ValueError)


# ------------------------------------------------- terrain, wind, padding
def test_slope_from_altitude_matches_reference():
    alt = np.load(gold("altitude.npy"))
    h = META["helpers"]
    assert sha(data_io.slope_from_altitude(alt, 25.0)) == h["slope_from_altitude"]
    assert sha(data_io.slope_from_altitude(alt, 25.0, "uphill-positive")) == \
        h["slope_from_altitude_uphill"]


def test_slope_known_values_and_errors():
    alt = np.array([[30.0, 0.0], [0.0, 0.0]])
    s = data_io.slope_from_altitude(alt, 30.0)
    assert s[0, 0, 1, 2] == pytest.approx(45.0)                # drop of one cell side
    assert s[0, 0, 2, 2] == pytest.approx(np.degrees(np.arctan(1 / np.sqrt(2))))
    assert s[0, 1, 1, 0] == -s[0, 0, 1, 2]                     # exact antisymmetry
    assert not s[:, :, 1, 1].any() and not s[0, :, 0, :].any()  # centre, off-grid
    with pytest.raises(ValueError, match="slope_sign"):
        data_io.slope_from_altitude(alt, 30.0, "sideways")
    with pytest.raises(ValueError, match="non-finite"):
        data_io.slope_from_altitude(np.array([[np.nan]]), 30.0)
    with pytest.raises(ValueError):
        data_io.slope_from_altitude(alt, 0.0)
    assert not data_io.slope_from_altitude(np.zeros((1, 1)), 30.0).any()


def test_wind_from_uv_matches_reference():
    u, v = np.load(gold("uv.npy"))
    s, d = data_io.wind_from_uv(u, v)
    assert [sha(s), sha(d)] == META["helpers"]["wind_from_uv"]
    assert ((d >= 0) & (d < 360)).all()
    s, d = data_io.wind_from_uv([0.0], [-2.0])
    assert s[0] == 2.0 and d[0] == 270.0
    with pytest.raises(ValueError, match="shape mismatch"):
        data_io.wind_from_uv(np.zeros(2), np.zeros(3))


def test_pad_nonburnable_matches_reference():
    pad = data_io.pad_nonburnable(synthetic.make_landscape("hill", 9), 2)
    assert {f: sha(getattr(pad, f)) for f in FIELDS} == META["helpers"]["pad_nonburnable"]
    land = synthetic.make_landscape("hill", 5)
    assert data_io.pad_nonburnable(land, 0) is land
    with pytest.raises(ValueError):
        data_io.pad_nonburnable(land, -1)


@pytest.mark.parametrize("key", sorted(META["landscapes"]))
def test_synthetic_landscapes_bit_identical(key):
    kind, sign = key.split("|")
    land = synthetic.make_landscape(kind, 17, slope_sign=sign)
    assert {f: sha(getattr(land, f)) for f in FIELDS} == META["landscapes"][key]


def test_unknown_synthetic_kind():
    with pytest.raises(ValueError, match="unknown synthetic landscape"):
        synthetic.make_landscape("volcano", 8)


# ------------------------------------------------------------------ bundles
@pytest.mark.parametrize("bundle,kind,sign", [("bundle_hill", "hill", "downhill-positive"),
                                              ("bundle_random", "random:5", "uphill-positive")])
def test_bundle_read_and_write(tmp_path, bundle, kind, sign):
    land = data_io.read_landscape(gold(bundle))
    src = synthetic.make_landscape(kind, land.height, slope_sign=sign)
    for f in FIELDS:
        assert getattr(land, f).dtype == np.float64
        assert np.array_equal(getattr(land, f), getattr(src, f).astype(np.float32))
    assert land.cell_side == 30.0
    data_io.write_landscape(src, tmp_path / "b")
    for name in os.listdir(gold(bundle)):
        assert (tmp_path / "b" / name).read_bytes() == open(gold(bundle, name), "rb").read()


def test_bundle_missing_grid_reported(tmp_path):
    data_io.write_landscape(synthetic.make_landscape("flat", 4), tmp_path)
    os.remove(tmp_path / "canopy.ptfg")
    with pytest.raises(FileNotFoundError, match="canopy.ptfg"):
        data_io.read_landscape(tmp_path)


def test_manifest_round_trip(tmp_path):
    entries = {"cell_side": "12.5", "note": "a=b"}
    data_io.write_manifest(entries, tmp_path / "m.txt")
    assert (tmp_path / "m.txt").read_text() == "cell_side=12.5\nnote=a=b\n"
    (tmp_path / "m.txt").write_text((tmp_path / "m.txt").read_text() + "# comment\n\n")
    assert data_io.read_manifest(tmp_path / "m.txt") == entries


# --------------------------------------------------------- snapshots/series
def test_render_state_matches_reference():
    burning, burned = np.load(gold("render_masks.npy"))
    st = FireState(burning, burned, np.zeros(burning.shape), 0)
    img = data_io.render_state(st, synthetic.make_landscape("random:4", 12))
    assert sha(img) == META["helpers"]["render_state"]
    r, c = np.argwhere(burning)[0]
    assert tuple(img[r, c]) == (255, 0, 0)


def test_snapshot_header(tmp_path):
    land = synthetic.make_landscape("flat", 3)
    st = FireState(np.eye(3, dtype=bool), np.zeros((3, 3), bool), np.zeros((3, 3)), 0)
    data_io.write_snapshot(st, land, tmp_path / "s.ppm")
    blob = (tmp_path / "s.ppm").read_bytes()
    assert blob.startswith(b"P6\n3 3\n255\n") and len(blob) == 11 + 27


def test_series_csv_forms(tmp_path):
    recs = [StepStats(t=1, burning=3, burned=1), StepStats(t=2, burning=2, burned=5)]
    data_io.write_series_csv(recs, tmp_path / "a.csv")
    data_io.write_series_csv(np.array([[3, 1], [2, 5]]), tmp_path / "b.csv")
    text = "step,burning,burned,affected\n1,3,1,4\n2,2,5,7\n"
    assert (tmp_path / "a.csv").read_bytes() == text.encode()
    assert (tmp_path / "b.csv").read_bytes() == text.encode()
    data_io.write_series_csv(recs, tmp_path / "j.csv", jaccard=[0.5, 1 / 3])
    assert (tmp_path / "j.csv").read_text().splitlines()[2] == "2,2,5,7,0.333333"
    with pytest.raises(ValueError, match="length mismatch"):
        data_io.write_series_csv(recs, tmp_path / "x.csv", jaccard=[0.5])
    data_io.write_series_csv([], tmp_path / "e.csv")
    assert (tmp_path / "e.csv").read_text() == "step,burning,burned,affected\n"


# --------------------------------------------------------- CLI (host side)
def test_cli_parser_mirrors_reference_flags():
    ap = cli.build_parser()
    a = ap.parse_args(["simulate", "--synthetic", "windy", "--size", "8", "--p-h", "0.4",
                       "--p-continue", "0.2", "--factor-site", "source", "--slope-units",
                       "radians", "--snapshot-every", "3", "--out", "o"])
    assert (a.p_h, a.p_continue, a.factor_site, a.slope_units, a.snapshot_every) == \
        (0.4, 0.2, "source", "radians", 3)
    b = ap.parse_args(["bench"])
    assert (b.sizes, b.steps, b.threads, b.seed) == ("200,400", 300, "1", 0)
    c = ap.parse_args(["calibrate", "--synthetic", "flat", "--target", "x", "--target", "y",
                       "--rings", "1,2,3", "--out", "o"])
    assert c.target == ["x", "y"] and c.rings == "1,2,3"


def test_cli_metrics_matches_reference(capsys):
    s = gold("sim_windy")
    code = cli.main(["metrics", "--pred", os.path.join(s, "affected_00006.ptfg"),
                     "--pred", os.path.join(s, "affected_00012.ptfg"),
                     "--target", os.path.join(s, "affected_00012.ptfg"),
                     "--target", os.path.join(s, "final_burning.ptfg")])
    assert code == 0
    assert capsys.readouterr().out == META["metrics_stdout"]


def test_cli_errors(tmp_path, capsys):
    with pytest.raises(SystemExit, match="need --landscape"):
        cli.main(["simulate", "--out", str(tmp_path / "o")])
    with pytest.raises(SystemExit, match="counts differ"):
        cli.main(["metrics", "--pred", "a", "--pred", "b", "--target", "c"])
    with pytest.raises(SystemExit, match="target"):
        cli.main(["calibrate", "--synthetic", "flat", "--size", "8", "--out", str(tmp_path)])
    g = gold("bool_2d.ptfg")
    with pytest.raises(SystemExit, match="shape mismatch"):
        cli.main(["metrics", "--pred", g, "--target", gold("f32_2d.ptfg")])
    # bundle problems surface as exit code 1 with the file named
    assert cli.main(["simulate", "--landscape", str(tmp_path / "nowhere"), "--out",
                     str(tmp_path / "o")]) == 1
    assert "wind_speed.ptfg" in capsys.readouterr().err


def test_cli_config_precedence():
    ap = cli.build_parser()
    a = ap.parse_args(["simulate", "--steps", "4", "--out", "o"])
    cfg = {"steps": "9", "seed": "11", "c1": "0.5"}
    assert cli._setting(a, cfg, "steps", int, 100) == 4
    assert cli._setting(a, cfg, "seed", int, 0) == 11
    assert cli._load_params(a, cfg).c1 == 0.5
