"""Seeded synthetic inputs for the BASELINE.json configs (c0..c4).

The paper's real datasets are absent, so every benchmark and parity case runs
on these generators.  The ambiguous points of the config text are frozen here
once and fed identically to the device path and the CPU
oracle:

* elevation: white noise U[0,1), periodic Gaussian smoothing (sigma cells),
  min-max rescaled to [0, 1500] m;
* wind speed: U[0,10] noise, periodic Gaussian smoothing, min-max rescaled
  back to [0, 10] m/s (smoothing alone collapses it to ~[4.9, 5.1]);
* wind direction: uniform angle, smoothed sin/cos components, atan2, degrees
  East-CCW in [0, 360) (the reference's convention, pyrocell/model.py:80);
* p_veg over {-0.3, 0, 0.4}, p_den over {-0.4, 0, 0.3}, both with
  probabilities {0.3, 0.4, 0.3};
* every field is rounded to fp32 (the configs say "fp32 grid"); the oracle
  and reference receive the same fp32 values promoted to fp64;
* slope for the reference API = slope_from_altitude(E, 30 m) downhill-positive
  (pyrocell/data_io.py:92-132); the device path derives it on the fly.

c0/c1/c2/c4 use scipy's gaussian_filter (mode="wrap", truncate 4) on the
host, which is deterministic across hosts with the same image.  c3
(16384^2, sigma x32) uses a periodic FFT Gaussian on the GPU because the
spatial filter is impractical there; no CPU golden depends on c3.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

VEG_VALUES = (-0.3, 0.0, 0.4)
DEN_VALUES = (-0.4, 0.0, 0.3)
CAT_PROBS = (0.3, 0.4, 0.3)
CELL_SIDE = 30.0

# (a, c1, c2, p_h, p_continue) used by every config unless stated otherwise
DEFAULT_BENCH_PARAMS = dict(a=0.078, c1=0.045, c2=0.131, p_h=0.58, p_continue=0.3)
HIDDEN_C2_PARAMS = dict(a=0.1, c1=0.06, c2=0.1, p_h=0.5, p_continue=0.35)


@dataclass
class Environment:
    """Host fp32 rasters of one landscape (elevation mode)."""

    elevation: np.ndarray       # (H, W) m
    wind_speed: np.ndarray      # (H, W) m/s
    wind_direction: np.ndarray  # (H, W) degrees East-CCW
    canopy: np.ndarray          # p_veg
    density: np.ndarray         # p_den
    cell_side: float = CELL_SIDE

    @property
    def shape(self) -> Tuple[int, int]:
        return self.elevation.shape

    def fingerprint(self) -> str:
        import hashlib
        h = hashlib.sha256()
        for a in (self.elevation, self.wind_speed, self.wind_direction, self.canopy,
                  self.density):
            h.update(np.ascontiguousarray(a, dtype=np.float32).tobytes())
        return h.hexdigest()[:16]


def _minmax(x: np.ndarray, lo: float, hi: float) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    mn, mx = float(x.min()), float(x.max())
    if mx <= mn:
        return np.full(x.shape, lo)
    return lo + (x - mn) * ((hi - lo) / (mx - mn))


def _smooth_host(x: np.ndarray, sigma: float) -> np.ndarray:
    from scipy.ndimage import gaussian_filter
    return gaussian_filter(x, sigma, mode="wrap")


def make_environment(h: int, w: Optional[int] = None, *, seed: int = 0,
                     sigma_elev: float = 20.0, sigma_wind: float = 30.0,
                     smoother=None) -> Environment:
    """Config-0 style environment at any size (c0/c1/c2/c4 use sigma 20/30)."""
    w = h if w is None else w
    smooth = smoother or _smooth_host
    rng = np.random.default_rng([seed, 0xE1E7])
    elev = _minmax(smooth(rng.random((h, w)), sigma_elev), 0.0, 1500.0)
    rng = np.random.default_rng([seed, 0x5EED])
    speed = _minmax(smooth(rng.uniform(0.0, 10.0, (h, w)), sigma_wind), 0.0, 10.0)
    rng = np.random.default_rng([seed, 0xD1EC])
    ang = rng.uniform(0.0, 2.0 * np.pi, (h, w))
    s, c = smooth(np.sin(ang), sigma_wind), smooth(np.cos(ang), sigma_wind)
    direction = np.mod(np.degrees(np.arctan2(s, c)), 360.0)
    rng = np.random.default_rng([seed, 0x7E6])
    veg = rng.choice(np.array(VEG_VALUES), size=(h, w), p=CAT_PROBS)
    rng = np.random.default_rng([seed, 0xDE5])
    den = rng.choice(np.array(DEN_VALUES), size=(h, w), p=CAT_PROBS)
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    direction = f32(direction)
    direction[direction >= 360.0] = 0.0  # fp32 rounding of values just below 360
    return Environment(f32(elev), f32(speed), direction, f32(veg), f32(den))


def center_ignition(h: int, w: Optional[int] = None, block: int = 3) -> np.ndarray:
    """block x block burning square at the grid centre (the semantics of
    pyrocell/synthetic.py:129-136, generalised to rectangles)."""
    w = h if w is None else w
    init = np.zeros((h, w), dtype=bool)
    half = block // 2
    r0 = max(h // 2 - half, 0)
    c0 = max(w // 2 - half, 0)
    init[r0:min(r0 + block, h), c0:min(c0 + block, w)] = True
    return init


def random_block_origins(h: int, w: int, n: int = 8, block: int = 5, seed: int = 3):
    """Top-left cells of random_blocks' ignitions."""
    rng = np.random.default_rng([seed, 0xB10C])
    rows = rng.integers(block, h - 2 * block, n)
    cols = rng.integers(block, w - 2 * block, n)
    return [(int(r), int(c)) for r, c in zip(rows, cols)]


def random_blocks(h: int, w: int, n: int = 8, block: int = 5, seed: int = 3) -> np.ndarray:
    """n randomly placed block x block ignitions (config 3)."""
    init = np.zeros((h, w), dtype=bool)
    for r, c in random_block_origins(h, w, n, block, seed):
        init[r:r + block, c:c + block] = True
    return init


def ensemble_ph(n_members: int, p_h: float = 0.58, seed: int = 1) -> np.ndarray:
    """Config 1: p_h jittered uniformly in +-10% per member."""
    rng = np.random.default_rng([seed, 0x9A])
    return p_h * rng.uniform(0.9, 1.1, n_members)


def reference_landscape_arrays(env: Environment, slope_fn):
    """fp64 arrays the reference API consumes (pyrocell Landscape fields),
    built from the fp32 environment; slope_fn is slope_from_altitude."""
    f64 = lambda a: np.asarray(a, dtype=np.float64)
    return dict(wind_speed=f64(env.wind_speed), wind_direction=f64(env.wind_direction),
                slope=slope_fn(f64(env.elevation), env.cell_side),
                canopy=f64(env.canopy), density=f64(env.density))


def fft_gaussian_torch(x, sigma: float):
    """Periodic Gaussian smoothing via FFT (torch, any device); used for c3."""
    import torch
    h, w = x.shape
    fy = torch.fft.fftfreq(h, device=x.device, dtype=torch.float64)
    fx = torch.fft.rfftfreq(w, device=x.device, dtype=torch.float64)
    g = torch.exp(-2.0 * (np.pi ** 2) * sigma ** 2 * (fy[:, None] ** 2 + fx[None, :] ** 2))
    X = torch.fft.rfft2(x.to(torch.float64))
    return torch.fft.irfft2(X * g, s=(h, w))


def make_environment_torch(h: int, w: int, *, seed: int = 0, sigma_elev: float = 640.0,
                           sigma_wind: float = 960.0, device="cuda") -> dict:
    """Config-3 environment generated on the device (fp32 tensors)."""
    import torch
    gen = torch.Generator(device=device)

    def rand(salt, lo=0.0, hi=1.0):
        gen.manual_seed(seed * 1000003 + salt)
        return lo + (hi - lo) * torch.rand((h, w), generator=gen, device=device,
                                           dtype=torch.float64)

    def mm(x, lo, hi):
        mn, mx = x.min(), x.max()
        return lo + (x - mn) * ((hi - lo) / (mx - mn))

    elev = mm(fft_gaussian_torch(rand(1), sigma_elev), 0.0, 1500.0)
    speed = mm(fft_gaussian_torch(rand(2, 0.0, 10.0), sigma_wind), 0.0, 10.0)
    ang = rand(3, 0.0, 2 * np.pi)
    s = fft_gaussian_torch(torch.sin(ang), sigma_wind)
    c = fft_gaussian_torch(torch.cos(ang), sigma_wind)
    direction = torch.remainder(torch.rad2deg(torch.atan2(s, c)), 360.0).float()
    direction[direction >= 360.0] = 0.0

    def cat(salt, values):
        u = rand(salt)
        v = torch.full((h, w), values[1], device=device, dtype=torch.float64)
        v[u < CAT_PROBS[0]] = values[0]
        v[u >= CAT_PROBS[0] + CAT_PROBS[1]] = values[2]
        return v.float()

    return dict(elevation=elev.float(), wind_speed=speed.float(), wind_direction=direction,
                canopy=cat(4, VEG_VALUES), density=cat(5, DEN_VALUES))


# ----------------------------------------------- named reference landscapes
# The generator kinds the reference CLI and tests use (pyrocell/synthetic.py:
# 13-126): host fp64 Landscapes with (H, W, 3, 3) slope grids.
def _box_smooth(grid: np.ndarray, passes: int) -> np.ndarray:
    """passes x 3x3 box mean with edge clamping (synthetic.py:13-23); the
    nine shifted views are summed in row-major offset order."""
    out = np.asarray(grid, dtype=np.float64)
    h, w = out.shape
    for _ in range(passes):
        p = np.pad(out, 1, mode="edge")
        acc = np.zeros_like(out)
        for dr in range(3):
            for dc in range(3):
                acc += p[dr:dr + h, dc:dc + w]
        out = acc / 9.0
    return out


def _dome(size: int, height_m: float) -> np.ndarray:
    t = np.linspace(-1.0, 1.0, size)
    x, y = np.meshgrid(t, t)
    return height_m * np.exp(-2.0 * (x * x + y * y))


def _land(speed, direction, altitude, canopy, density, cell_side, slope_sign):
    from .data_io import slope_from_altitude
    from .model import Landscape
    size = np.shape(canopy)[0]
    full = lambda v: np.full((size, size), float(v)) if np.isscalar(v) else np.asarray(v, np.float64)
    slope = (np.zeros((size, size, 3, 3)) if altitude is None
             else slope_from_altitude(altitude, cell_side, slope_sign))
    return Landscape(wind_speed=full(speed), wind_direction=full(direction), slope=slope,
                     canopy=full(canopy), density=full(density), cell_side=cell_side)


def flat_landscape(size: int, cell_side: float = 30.0):
    """Windless plain, neutral vegetation."""
    z = np.zeros((size, size))
    return _land(0.0, 0.0, None, z, z, cell_side, "downhill-positive")


def hill_landscape(size: int, cell_side: float = 30.0, slope_sign: str = "downhill-positive"):
    """Dome of 8 cell sides, 3 m/s toward 45 degrees."""
    z = np.zeros((size, size))
    return _land(3.0, 45.0, _dome(size, 8.0 * cell_side), z, z, cell_side, slope_sign)


def valley_landscape(size: int, cell_side: float = 30.0, slope_sign: str = "downhill-positive"):
    """Inverted dome, 3 m/s toward 225 degrees."""
    z = np.zeros((size, size))
    return _land(3.0, 225.0, -_dome(size, 8.0 * cell_side), z, z, cell_side, slope_sign)


def windy_landscape(size: int, cell_side: float = 30.0, slope_sign: str = "downhill-positive"):
    """Gentle dome (2 cell sides), 10 m/s toward 30 degrees, damped
    vegetation (canopy = density = -0.45)."""
    damp = np.full((size, size), -0.45)
    return _land(10.0, 30.0, _dome(size, 2.0 * cell_side), damp, damp, cell_side, slope_sign)


def random_landscape(size: int, seed: int, cell_side: float = 30.0,
                     slope_sign: str = "downhill-positive"):
    """Box-smoothed random terrain, wind and vegetation; draws in the order
    altitude, speed, direction, canopy, density from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    draw = lambda lo, hi: rng.uniform(lo, hi, (size, size))
    altitude = _box_smooth(draw(0.0, 6.0 * cell_side), 3)
    speed = np.clip(_box_smooth(draw(0.0, 6.0), 2), 0.0, None)
    direction = _box_smooth(draw(0.0, 360.0), 2) % 360.0
    canopy = np.clip(_box_smooth(draw(-0.4, 0.4), 2), -1.0, None)
    density = np.clip(_box_smooth(draw(-0.4, 0.4), 2), -1.0, None)
    return _land(speed, direction, altitude, canopy, density, cell_side, slope_sign)


def make_landscape(kind: str, size: int, cell_side: float = 30.0,
                   slope_sign: str = "downhill-positive"):
    """flat | hill | valley | windy | random:<seed> (synthetic.py:112-126)."""
    if kind == "flat":
        return flat_landscape(size, cell_side)
    makers = {"hill": hill_landscape, "valley": valley_landscape, "windy": windy_landscape}
    if kind in makers:
        return makers[kind](size, cell_side, slope_sign)
    if kind.startswith("random:"):
        return random_landscape(size, int(kind.split(":", 1)[1]), cell_side, slope_sign)
    raise ValueError(f"unknown synthetic landscape {kind!r}")
