"""ctypes front-end of the CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this
module; it is the checker and the CPU baseline, never the product path.

It restates the reference (pyrocell 0.1.0, pure NumPy) hot path:
  rng.py:35-88         -> uniform_grid, uniform_draw, derive_epoch_seed
  data_io.py:92-132    -> slope_from_altitude
  kernel.py:149-529    -> run (run_simulation + step_forward + tape record)
  tape.py:19-39        -> attachment_plan
  tape.py:118-148      -> contract (backward_params, per-cell Jacobian form)
  losses.py:44-86      -> combined_loss
  calibration.py:43-64 -> adamw_update
Pinned by tests/golden/ (vectors from the reference's own tests and from
running the reference itself, see tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

DEFAULT_NORM_C = 1.1486328125


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
                os.path.join(_HERE, "oracle.c")):
            build()
        L = C.CDLL(_SO)
        u64, i64, dp = C.c_uint64, C.c_int64, C.POINTER(C.c_double)
        L.orc_stream_key.restype = u64
        L.orc_stream_key.argtypes = [u64, u64, u64]
        L.orc_epoch_seed.restype = u64
        L.orc_epoch_seed.argtypes = [u64, u64]
        L.orc_uniform_grid.restype = None
        L.orc_uniform_grid.argtypes = [u64, u64, u64, i64, i64, i64, i64, C.c_void_p]
        L.orc_slope_from_altitude.restype = C.c_int
        L.orc_slope_from_altitude.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double,
                                              C.c_int, C.c_void_p]
        L.orc_run.restype = C.c_int
        L.orc_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, u64, C.c_int, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_combined_loss.restype = C.c_int
        L.orc_combined_loss.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                        C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_contract.restype = None
        L.orc_contract.argtypes = [C.c_void_p, C.c_void_p, i64, dp]
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------ RNG ---
IGNITE, CONTINUE = 0, 1


def uniform_grid(seed, t, channel, row0, col0, height, width) -> np.ndarray:
    out = np.empty((height, width), dtype=np.float64)
    lib().orc_uniform_grid(int(seed) & (2**64 - 1), int(t) & (2**64 - 1), int(channel),
                           row0, col0, height, width, _ptr(out))
    return out


def uniform_draw(seed, t, row, col, channel) -> float:
    return float(uniform_grid(seed, t, channel, row, col, 1, 1)[0, 0])


def derive_epoch_seed(base_seed: int, epoch: int) -> int:
    return int(lib().orc_epoch_seed(int(base_seed) & (2**64 - 1), int(epoch) & (2**64 - 1)))


# ---------------------------------------------------------------- slope ---
def slope_from_altitude(altitude, cell_side=30.0, slope_sign="downhill-positive") -> np.ndarray:
    e = np.ascontiguousarray(altitude, dtype=np.float64)
    h, w = e.shape
    out = np.empty((h, w, 3, 3), dtype=np.float64)
    rc = lib().orc_slope_from_altitude(_ptr(e), h, w, float(cell_side),
                                       int(slope_sign == "uphill-positive"), _ptr(out))
    if rc != 0:
        raise ValueError("cell_side must be > 0")
    return out


# ------------------------------------------------------------------ run ---
class _Model(C.Structure):
    _fields_ = [("h", C.c_int), ("w", C.c_int),
                ("vw", C.c_void_p), ("wdir", C.c_void_p), ("slope9", C.c_void_p),
                ("canopy", C.c_void_p), ("density", C.c_void_p),
                ("c1", C.c_double), ("c2", C.c_double), ("a", C.c_double),
                ("p_h", C.c_double), ("p_continue", C.c_double), ("norm_c", C.c_double),
                ("factor_source", C.c_int), ("slope_radians", C.c_int),
                ("row0", C.c_int64), ("col0", C.c_int64), ("wsched", C.c_void_p)]


@dataclass
class OracleResult:
    burning: np.ndarray
    burned: np.ndarray
    acc: np.ndarray
    t_ign: np.ndarray
    jac: Optional[np.ndarray]
    series: np.ndarray       # (steps, 2): burning, burned after each step
    n_entries: int
    jac_abs: Optional[np.ndarray] = None    # sum of |slot terms| per J component
    jac_floor: Optional[np.ndarray] = None  # rounding floor of the reference's own J
    jac_cond: Optional[np.ndarray] = None   # conditioning of an fp32 evaluation of J

    def affected(self):
        return self.burning | self.burned


def run(wind_speed, wind_direction, slope, canopy, density, params, init, steps, seed, *,
        attach_steps=(), wind_schedule=(), norm_c=DEFAULT_NORM_C, factor_site="target",
        slope_units="degrees", threads=1, want_jac=None, origin=(0, 0), wind_params=None,
        want_jac_abs=False) -> OracleResult:
    """Restates run_simulation (kernel.py:453-529).

    params: object with c1, c2, a, p_h, p_continue (floats).
    wind_schedule: iterable of (apply_at_step, speed, direction).
    origin: absolute (row, col) of local cell (0, 0) -- the arrays are a crop
    of a larger domain, draws keyed by the absolute cell (rng.py:64-67).
    wind_params: optional (steps, >=3) rows (alpha, beta, gamma_deg) per
    pre-step index: step t runs on the WindUpdate fields alpha*V + beta,
    theta + gamma of the base fields (the parametric form of kernel.py:505-511).
    """
    f64 = lambda x: np.ascontiguousarray(x, dtype=np.float64)
    vw, wd, sl, ca, de = f64(wind_speed), f64(wind_direction), f64(slope), f64(canopy), f64(density)
    h, w = vw.shape
    init_u8 = np.ascontiguousarray(np.asarray(init, dtype=bool).astype(np.uint8))
    sched = sorted(wind_schedule, key=lambda u: u[0])
    n_wind = len(sched)
    wind_at = np.array([int(u[0]) for u in sched] or [0], dtype=np.int32)
    wv = f64(np.stack([u[1] for u in sched])) if n_wind else np.zeros(1)
    wdd = f64(np.stack([u[2] for u in sched])) if n_wind else np.zeros(1)
    attach = np.zeros(steps + 1, dtype=np.uint8)
    for s in attach_steps:
        if 1 <= int(s) <= steps:
            attach[int(s)] = 1
    if want_jac is None:
        want_jac = bool(attach.any())
    wp = None
    if wind_params is not None:
        wp = np.zeros((max(steps, 1), 4), np.float64)
        src = np.asarray(wind_params, dtype=np.float64)
        wp[:min(steps, len(src)), :3] = src[:steps, :3]
    m = _Model(h, w, vw.ctypes.data, wd.ctypes.data, sl.ctypes.data, ca.ctypes.data,
               de.ctypes.data, float(params.c1), float(params.c2), float(params.a),
               float(params.p_h), float(params.p_continue), float(norm_c),
               int(factor_site == "source"), int(slope_units == "radians"),
               int(origin[0]), int(origin[1]), None if wp is None else wp.ctypes.data)
    burning = np.empty((h, w), np.uint8)
    burned = np.empty((h, w), np.uint8)
    acc = np.empty((h, w), np.float64)
    t_ign = np.empty((h, w), np.int32)
    jac = np.empty((h, w, 4), np.float64) if want_jac else None
    jac_abs = np.empty((h, w, 4), np.float64) if (want_jac and want_jac_abs) else None
    jac_floor = np.empty((h, w, 4), np.float64) if (want_jac and want_jac_abs) else None
    jac_cond = np.empty((h, w, 4), np.float64) if (want_jac and want_jac_abs) else None
    series = np.zeros((max(steps, 0), 2), np.int64)
    n_ent = C.c_int64(0)
    rc = lib().orc_run(C.byref(m), _ptr(init_u8), int(steps), int(seed) & (2**64 - 1), n_wind,
                       _ptr(wind_at), _ptr(wv), _ptr(wdd), _ptr(attach), int(threads),
                       _ptr(burning), _ptr(burned), _ptr(acc), _ptr(t_ign), _ptr(jac),
                       _ptr(jac_abs), _ptr(jac_floor), _ptr(jac_cond), _ptr(series),
                       C.byref(n_ent))
    if rc != 0:
        raise ValueError(f"oracle run failed ({rc})")
    return OracleResult(burning.astype(bool), burned.astype(bool), acc, t_ign, jac, series,
                        int(n_ent.value), jac_abs, jac_floor, jac_cond)


# ----------------------------------------------------------- tape/loss ---
def attachment_plan(total_steps: int, r_first: int, r_between: int, r_last: int):
    """Restates tape.py:19-39 (np.round is half-to-even)."""
    if total_steps < 0:
        raise ValueError("total_steps must be >= 0")
    att = set(range(1, min(r_first, total_steps) + 1))
    att.update(range(max(total_steps - r_last, 0) + 1, total_steps + 1))
    if r_between > 0:
        lo, hi = r_first + 1, total_steps - r_last + 1
        if hi > lo:
            for s in np.round(np.linspace(lo, hi, r_between + 2)[1:-1]).astype(int):
                if 1 <= s <= total_steps:
                    att.add(int(s))
    return tuple(sorted(att))


def combined_loss(acc, target):
    """Restates losses.py:44-86 -> (bce, mse, crop, grad)."""
    a = np.ascontiguousarray(acc, dtype=np.float64)
    y = np.ascontiguousarray(np.asarray(target, dtype=bool).astype(np.uint8))
    h, w = a.shape
    grad = np.empty((h, w), np.float64)
    terms = np.zeros(2, np.float64)
    crop = np.zeros(4, np.int32)
    lib().orc_combined_loss(_ptr(a), _ptr(y), h, w, _ptr(grad), _ptr(terms), _ptr(crop))
    return float(terms[0]), float(terms[1]), tuple(int(v) for v in crop), grad


def contract(jac, g) -> np.ndarray:
    """sum_j g_j J_j -> (dc1, dc2, da, dp_h); tape.py:118-148 per-cell form."""
    j = np.ascontiguousarray(jac, dtype=np.float64).reshape(-1, 4)
    gg = np.ascontiguousarray(g, dtype=np.float64).reshape(-1)
    out = (C.c_double * 4)()
    lib().orc_contract(_ptr(j), _ptr(gg), gg.size, out)
    return np.array(list(out))


def multi_target_grad(res: OracleResult, obs_steps: Sequence[int], targets):
    """Loss summed over observation steps of one run: acc_s = acc where the
    cell ignited before step s, grad via the Jacobian."""
    total, g = 0.0, np.zeros(res.acc.shape)
    for s, tgt in zip(obs_steps, targets):
        acc_s = np.where(res.t_ign < s, res.acc, 0.0)
        bce, mse, _, gs = combined_loss(acc_s, tgt)
        total += bce + mse
        g += np.where(res.t_ign < s, gs, 0.0)
    return total, contract(res.jac, g)


def adamw_update(state: dict, theta: np.ndarray, grads: np.ndarray, lr: float,
                 wd: float = 0.0, b1=0.9, b2=0.999, eps=1e-8) -> np.ndarray:
    """Restates calibration.py:43-64 on (c1, c2, a, p_h)."""
    grads = np.asarray(grads, dtype=np.float64)
    if not np.all(np.isfinite(grads)):
        raise ValueError(f"non-finite gradient: {grads}")
    state["t"] = state.get("t", 0) + 1
    state["m"] = b1 * state.get("m", np.zeros(4)) + (1 - b1) * grads
    state["v"] = b2 * state.get("v", np.zeros(4)) + (1 - b2) * grads * grads
    mh = state["m"] / (1 - b1 ** state["t"])
    vh = state["v"] / (1 - b2 ** state["t"])
    return theta - lr * (mh / (np.sqrt(vh) + eps) + wd * theta)
