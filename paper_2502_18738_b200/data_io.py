"""Raster I/O around the device path.

The module keeps the reference's name and public functions
(pyrocell/data_io.py) so ``from pyrocell import data_io`` callers switch by
changing the package name; the ``*_device`` functions are the B200 additions
that move payloads between files and device memory through pinned staging.

Grid container (data_io.py:16-89, "PTFG"): magic ``PTFG``, uint16 version 1,
uint8 dtype code (0 = little-endian float32, 1 = one byte per boolean cell),
uint8 rank, ``rank`` uint32 little-endian dims, row-major payload.  Errors
and their messages are the reference's (GridFileError and subclasses).

Landscape bundle (data_io.py:170-219): one PTFG grid per raster plus a
``key=value`` manifest.txt carrying cell_side.  ``read_landscape_device``
builds the kernel-layout ``DeviceLandscape`` (slope-tensor mode) straight
from the files without materialising the fp64 host Landscape.

Series CSV (data_io.py:244-262) and PPM snapshots (data_io.py:209-241) are
emitted from the per-step counters and bit planes the device keeps.
"""
from __future__ import annotations

import math
import struct
from pathlib import Path
from typing import Dict, Optional, Sequence, Tuple, Union

import numpy as np
import torch

from .device import NEIGHBOR_POSITIONS, DeviceLandscape, _dev
from .model import FireState, Landscape

MAGIC = b"PTFG"
FORMAT_VERSION = 1
_DTYPE_FLOAT32 = 0
_DTYPE_BOOL = 1
_BUNDLE_GRIDS = ("wind_speed", "wind_direction", "slope", "canopy", "density")

PathLike = Union[str, Path]


class GridFileError(ValueError):
    """Malformed or unsupported grid file (data_io.py:27-41)."""


class BadMagicError(GridFileError):
    pass


class TruncatedPayloadError(GridFileError):
    pass


class UnsupportedDtypeError(GridFileError):
    pass


# ------------------------------------------------------------------- header
def _header(code: int, shape: Sequence[int]) -> bytes:
    return MAGIC + struct.pack("<HBB", FORMAT_VERSION, code, len(shape)) + \
        struct.pack(f"<{len(shape)}I", *shape)


def _parse(blob: bytes, path) -> Tuple[int, Tuple[int, ...], int]:
    """(dtype code, dims, payload offset) of a PTFG blob, with the
    reference's checks in its order (data_io.py:63-89)."""
    if len(blob) < 8 or blob[:4] != MAGIC:
        raise BadMagicError(f"{path}: not a PTFG grid file")
    version, code, rank = struct.unpack("<HBB", blob[4:8])
    if version != FORMAT_VERSION:
        raise GridFileError(f"{path}: unsupported version {version}")
    if code not in (_DTYPE_FLOAT32, _DTYPE_BOOL):
        raise UnsupportedDtypeError(f"{path}: unknown dtype code {code}")
    end = 8 + 4 * rank
    if len(blob) < end:
        raise TruncatedPayloadError(f"{path}: truncated header")
    dims = struct.unpack(f"<{rank}I", blob[8:end])
    count = 1
    for d in dims:
        count *= d
    expected = count * (4 if code == _DTYPE_FLOAT32 else 1)
    if len(blob) - end != expected:
        raise TruncatedPayloadError(
            f"{path}: payload {len(blob) - end} bytes, expected {expected}")
    return code, tuple(dims), end


# --------------------------------------------------------------------- host
def write_grid(grid, path: PathLike) -> None:
    """data_io.py:43-60: float or integer grids as little-endian float32,
    booleans as one byte per cell; rank >= 1."""
    arr = np.asarray(grid)
    if arr.ndim < 1:
        raise GridFileError("grid must have rank >= 1")
    if arr.dtype == bool:
        code, payload = _DTYPE_BOOL, arr.astype(np.uint8).tobytes(order="C")
    elif np.issubdtype(arr.dtype, np.floating) or np.issubdtype(arr.dtype, np.integer):
        code, payload = _DTYPE_FLOAT32, arr.astype("<f4").tobytes(order="C")
    else:
        raise UnsupportedDtypeError(f"cannot store dtype {arr.dtype}")
    Path(path).write_bytes(_header(code, arr.shape) + payload)


def read_grid(path: PathLike) -> np.ndarray:
    """data_io.py:63-89: bit-exact inverse of write_grid (float32 or bool)."""
    blob = Path(path).read_bytes()
    code, dims, off = _parse(blob, path)
    if code == _DTYPE_FLOAT32:
        return np.frombuffer(blob, dtype="<f4", offset=off).reshape(dims).copy()
    return np.frombuffer(blob, dtype=np.uint8, offset=off).reshape(dims).astype(bool)


# ------------------------------------------------------------------- device
def read_grid_device(path: PathLike, device=None) -> torch.Tensor:
    """A PTFG grid as a device tensor: float32, or uint8 0/1 for a boolean
    grid (any non-zero byte reads as 1, like read_grid's astype(bool)).  The
    payload goes file -> pinned staging -> HBM in one copy."""
    dev = _dev(device)
    blob = Path(path).read_bytes()
    code, dims, off = _parse(blob, path)
    nbytes = len(blob) - off
    stage = torch.empty((nbytes,), dtype=torch.uint8, pin_memory=True)
    if nbytes:
        stage.numpy()[:] = np.frombuffer(blob, dtype=np.uint8, offset=off)
    dt = torch.float32 if code == _DTYPE_FLOAT32 else torch.uint8
    out = torch.empty(dims, dtype=dt, device=dev)
    out.view(torch.uint8).reshape(-1).copy_(stage, non_blocking=True)
    if code == _DTYPE_BOOL:
        out = (out != 0).to(torch.uint8)
    torch.cuda.current_stream(dev).synchronize()  # the staging buffer dies on return
    return out


def write_grid_device(t: torch.Tensor, path: PathLike, boolean: Optional[bool] = None) -> None:
    """A device tensor as a PTFG grid.  bool / uint8 tensors are written as
    boolean grids unless boolean=False; everything else as float32 (the
    fp64 accumulator is rounded like write_grid's astype('<f4'))."""
    if t.dim() < 1:
        raise GridFileError("grid must have rank >= 1")
    is_bool = boolean if boolean is not None else t.dtype in (torch.bool, torch.uint8)
    if is_bool:
        src, code = (t != 0).to(torch.uint8).contiguous(), _DTYPE_BOOL
    else:
        src, code = t.to(torch.float32).contiguous(), _DTYPE_FLOAT32
    stage = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
    stage.copy_(src, non_blocking=True)
    torch.cuda.current_stream(src.device).synchronize()
    Path(path).write_bytes(_header(code, tuple(src.shape)) + stage.numpy().tobytes(order="C"))


# ------------------------------------------------------- terrain and wind
def slope_from_altitude(altitude, cell_side: float,
                        slope_sign: str = "downhill-positive") -> np.ndarray:
    """data_io.py:92-132: (H, W, 3, 3) degrees from each cell toward each
    neighbour, atan((E_i - E_j) / (k * cell_side)) with k = sqrt(2) on
    diagonals; off-grid neighbours and the centre are 0; the reverse
    direction of every pair is the exact negation.  uphill-positive negates
    the grid."""
    e = np.asarray(altitude, dtype=np.float64)
    if e.ndim != 2:
        raise ValueError(f"altitude must be 2-D, got shape {e.shape}")
    if not np.all(np.isfinite(e)):
        raise ValueError("altitude contains non-finite values")
    if cell_side <= 0:
        raise ValueError("cell_side must be > 0")
    if slope_sign not in ("downhill-positive", "uphill-positive"):
        raise ValueError(f"unknown slope_sign {slope_sign!r}")
    h, w = e.shape
    out = np.zeros((h, w, 3, 3), dtype=np.float64)
    for dr, dc in ((0, 1), (1, -1), (1, 0), (1, 1)):   # E, SW, S, SE
        dist = (math.sqrt(2.0) if dr and dc else 1.0) * cell_side
        rs, re_ = max(-dr, 0), h - max(dr, 0)
        cs, ce = max(-dc, 0), w - max(dc, 0)
        if re_ <= rs or ce <= cs:
            continue
        a = e[rs:re_, cs:ce]
        b = e[rs + dr:re_ + dr, cs + dc:ce + dc]
        deg = np.degrees(np.arctan((a - b) / dist))
        out[rs:re_, cs:ce, 1 + dr, 1 + dc] = deg
        out[rs + dr:re_ + dr, cs + dc:ce + dc, 1 - dr, 1 - dc] = -deg
    return -out if slope_sign == "uphill-positive" else out


def wind_from_uv(u, v) -> Tuple[np.ndarray, np.ndarray]:
    """data_io.py:135-145: (speed, direction degrees East-CCW in [0, 360))."""
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if u.shape != v.shape:
        raise ValueError(f"shape mismatch: {u.shape} vs {v.shape}")
    return np.hypot(u, v), np.degrees(np.arctan2(v, u)) % 360.0


def pad_nonburnable(land: Landscape, pad: int) -> Landscape:
    """data_io.py:148-173: a border of cells with canopy = density = -1
    (vd = 0, never ignite), zero wind and slope."""
    if pad < 0:
        raise ValueError("pad must be >= 0")
    if pad == 0:
        return land
    p2 = ((pad, pad), (pad, pad))
    return Landscape(
        wind_speed=np.pad(land.wind_speed, p2, constant_values=0.0),
        wind_direction=np.pad(land.wind_direction, p2, constant_values=0.0),
        slope=np.pad(land.slope, p2 + ((0, 0), (0, 0)), constant_values=0.0),
        canopy=np.pad(land.canopy, p2, constant_values=-1.0),
        density=np.pad(land.density, p2, constant_values=-1.0),
        cell_side=land.cell_side)


# ------------------------------------------------------------------ bundles
def write_manifest(entries: Dict[str, str], path: PathLike) -> None:
    Path(path).write_text("\n".join(f"{k}={v}" for k, v in entries.items()) + "\n")


def read_manifest(path: PathLike) -> Dict[str, str]:
    entries: Dict[str, str] = {}
    for line in Path(path).read_text().splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, _, value = line.partition("=")
        entries[key.strip()] = value.strip()
    return entries


def _bundle_paths(directory: PathLike):
    src = Path(directory)
    paths = {}
    for name in _BUNDLE_GRIDS:
        p = src / f"{name}.ptfg"
        if not p.exists():
            raise FileNotFoundError(f"landscape bundle missing grid: {p}")
        paths[name] = p
    manifest = read_manifest(src / "manifest.txt") if (src / "manifest.txt").exists() else {}
    return paths, float(manifest.get("cell_side", 30.0))


def write_landscape(land: Landscape, directory: PathLike) -> None:
    """data_io.py:192-197."""
    out = Path(directory)
    out.mkdir(parents=True, exist_ok=True)
    for name in _BUNDLE_GRIDS:
        write_grid(getattr(land, name), out / f"{name}.ptfg")
    write_manifest({"cell_side": repr(land.cell_side)}, out / "manifest.txt")


def read_landscape(directory: PathLike) -> Landscape:
    """data_io.py:200-219: the host Landscape (fp64 rasters)."""
    paths, cell_side = _bundle_paths(directory)
    grids = {k: read_grid(p).astype(np.float64) for k, p in paths.items()}
    return Landscape(cell_side=cell_side, **grids)


def read_landscape_device(directory: PathLike, *, factor_site: str = "target",
                          slope_units: str = "degrees", device=None) -> DeviceLandscape:
    """A bundle straight into the kernel layout on the device: the same
    landscape as DeviceLandscape.from_slope_tensor(read_landscape(dir)) --
    float32 payloads widen exactly, as read_landscape's astype(float64) does
    -- with the (H, W, 3, 3) slope regrouped into the per-slot source-side
    [H][W][8] tensor on the device instead of on the host."""
    if slope_units not in ("degrees", "radians"):
        raise ValueError(f"slope_units must be 'degrees' or 'radians', got {slope_units!r}")
    dev = _dev(device)
    paths, cell_side = _bundle_paths(directory)
    g = {k: read_grid_device(p, dev) for k, p in paths.items()}
    g = {k: (t.to(torch.float32) if t.dtype == torch.uint8 else t) for k, t in g.items()}
    sl = g["slope"]
    if sl.dim() != 4 or tuple(sl.shape[2:]) != (3, 3):
        raise ValueError(f"bundle slope must be (H, W, 3, 3), got {tuple(sl.shape)}")
    sl = sl.to(torch.float64)
    if slope_units == "radians":
        sl = torch.rad2deg(sl)
    h, w = sl.shape[:2]
    for name in ("wind_speed", "wind_direction", "canopy", "density"):
        if tuple(g[name].shape) != (h, w):
            raise ValueError(f"{name} shape {tuple(g[name].shape)} != {(h, w)}")
    # slot k at the source: slope toward the target = source - position
    s8 = torch.stack([sl[:, :, 1 - pr, 1 - pc] for pr, pc in NEIGHBOR_POSITIONS], dim=-1)
    zeros = torch.zeros((h, w), dtype=torch.float32, device=dev)
    land = DeviceLandscape.from_elevation(zeros, g["wind_speed"], g["wind_direction"],
                                          g["canopy"], g["density"], cell_side=cell_side,
                                          factor_site=factor_site, device=dev)
    land.slope64 = s8.contiguous()
    land.slope32 = land.slope64.to(torch.float32)
    return land


# ---------------------------------------------------- snapshots and series
_COLOR_BURNING = (255, 0, 0)
_COLOR_BURNED = (0, 0, 0)
_COLOR_SPARSE = np.array((150, 40, 170), dtype=np.float64)
_COLOR_DENSE = np.array((40, 170, 60), dtype=np.float64)


def render_state(state: FireState, land: Landscape) -> np.ndarray:
    """data_io.py:222-231: (H, W, 3) uint8 -- vegetation/steepness shade
    (purple sparse/gentle -> green dense/steep), burned black, burning red."""
    veg = np.clip(((land.canopy + land.density) / 2.0 + 1.0) / 2.0, 0.0, 1.0)
    steep = np.clip(np.mean(np.abs(land.slope), axis=(2, 3)) / 45.0, 0.0, 1.0)
    mix = np.clip(0.5 * veg + 0.5 * steep, 0.0, 1.0)[..., None]
    img = np.clip(_COLOR_SPARSE + mix * (_COLOR_DENSE - _COLOR_SPARSE), 1, 254).astype(np.uint8)
    img[state.burned] = _COLOR_BURNED
    img[state.burning] = _COLOR_BURNING
    return img


def write_snapshot(state: FireState, land: Landscape, path: PathLike) -> None:
    """data_io.py:234-241: binary PPM (P6), deterministic bytes."""
    img = render_state(state, land)
    h, w, _ = img.shape
    Path(path).write_bytes(f"P6\n{w} {h}\n255\n".encode("ascii") + img.tobytes(order="C"))


def _series_rows(series):
    """(t, burning, burned, affected) rows from StepStats records or from a
    (steps, 2) array of (burning, burned) device counters (t = 1..steps)."""
    if isinstance(series, (np.ndarray, torch.Tensor)):
        ser = np.asarray(series.cpu() if torch.is_tensor(series) else series, dtype=np.int64)
        return [(i + 1, int(b), int(d), int(b) + int(d)) for i, (b, d) in enumerate(ser)]
    return [(s.t, s.burning, s.burned, s.affected) for s in series]


def write_series_csv(series, path: PathLike, jaccard: Optional[Sequence[float]] = None) -> None:
    """data_io.py:244-262: step,burning,burned,affected[,jaccard], LF
    endings.  ``series`` is the reference's StepStats list or the
    FireBatch.series() counters of one member."""
    rows = _series_rows(series)
    if jaccard is not None and len(jaccard) != len(rows):
        raise ValueError("jaccard series length mismatch")
    lines = ["step,burning,burned,affected" + (",jaccard" if jaccard is not None else "")]
    for i, (t, b, d, a) in enumerate(rows):
        lines.append(f"{t},{b},{d},{a}" + (f",{jaccard[i]:.6f}" if jaccard is not None else ""))
    Path(path).write_bytes(("\n".join(lines) + "\n").encode("ascii"))
