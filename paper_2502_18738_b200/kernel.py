"""Forward CA API with the reference's signatures (pyrocell/kernel.py).

run_simulation / step_forward keep the reference's arguments, validation,
exceptions and results (host NumPy in and out) while every step runs in the
sm_100a step kernel (libfirecell fc_run) on device-resident bit planes.
The scalar helpers (wind_factor ... ignition_prob) are the closed-form
semantics the reference exposes for its tests; they are host formulas, not
the hot path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np
import torch

from .device import DEFAULT_NORM_C, NEIGHBOR_POSITIONS, DeviceLandscape, FireBatch, \
    build_fields_device, pack_params
from .model import FireState, Landscape, ModelParams, new_fire_state
from .tape import RunBinding, Tape

# kernel.py:38-47
OFFSET_BEARINGS = {
    (0, 1): 0.0, (-1, 1): 45.0, (-1, 0): 90.0, (-1, -1): 135.0,
    (0, -1): 180.0, (1, -1): 225.0, (1, 0): 270.0, (1, 1): 315.0,
}
PROPAGATION_BEARINGS = tuple(OFFSET_BEARINGS[(-pr, -pc)] for pr, pc in NEIGHBOR_POSITIONS)


# ------------------------------------------------------ scalar semantics ---
def wind_factor(c1: float, c2: float, v_w: float, theta_rel_deg: float) -> float:
    """kernel.py:50-58 (Eq. 2-3)."""
    return math.exp(c1 * v_w) * math.exp(c2 * v_w * (math.cos(math.radians(theta_rel_deg)) - 1.0))


def slope_factor(a: float, theta_s_deg: float) -> float:
    """kernel.py:61-63 (Eq. 4)."""
    return math.exp(a * theta_s_deg)


def propagate_prob(params: ModelParams, land: Landscape, from_cell, to_cell,
                   factor_site: str = "target") -> float:
    """kernel.py:66-94 (Eq. 5): raw spread factor from from_cell to to_cell."""
    fr, fc = from_cell
    tr, tc = to_cell
    off = (tr - fr, tc - fc)
    if off not in OFFSET_BEARINGS:
        raise ValueError(f"{to_cell} is not a Moore neighbor of {from_cell}")
    site = (tr, tc) if factor_site == "target" else (fr, fc)
    rel = float(land.wind_direction[fr, fc]) - OFFSET_BEARINGS[off]
    return (params.p_h * (1.0 + float(land.canopy[site])) * (1.0 + float(land.density[site]))
            * wind_factor(params.c1, params.c2, float(land.wind_speed[fr, fc]), rel)
            * slope_factor(params.a, float(land.slope[fr, fc, 1 + off[0], 1 + off[1]])))


def normalize_prob(x, c: float = DEFAULT_NORM_C):
    """kernel.py:97-99 (Eq. 9 normalisation)."""
    return np.tanh(c * x)


def ignition_prob(neighbor_probs: Sequence[float]) -> float:
    """kernel.py:102-114: 1 - prod(1 - p_i) in the caller's order."""
    probs = list(neighbor_probs)
    if not probs:
        return 0.0
    if len(probs) == 1:
        return float(probs[0])
    q = 1.0
    for p in probs:
        q *= 1.0 - p
    return 1.0 - q


# ------------------------------------------------------------- records ---
@dataclass
class PropagationFields:
    """kernel.py:128-146."""

    fp: np.ndarray
    vw: np.ndarray
    raw: Optional[np.ndarray] = None
    rest: Optional[np.ndarray] = None
    cosm1: Optional[np.ndarray] = None
    slope_toward: Optional[np.ndarray] = None
    site_is_target: bool = True

    @property
    def has_gradients(self) -> bool:
        return self.raw is not None


@dataclass(frozen=True)
class WindUpdate:
    """kernel.py:422-428."""

    apply_at_step: int
    wind_speed: np.ndarray
    wind_direction: np.ndarray


@dataclass
class StepStats:
    """kernel.py:431-439."""

    t: int
    burning: int
    burned: int

    @property
    def affected(self) -> int:
        return self.burning + self.burned


@dataclass
class SimulationResult:
    """kernel.py:442-450."""

    state: FireState
    series: List[StepStats]
    snapshots: List[Tuple[int, FireState]]
    tape: Optional[Tape] = None

    def affected_counts(self) -> List[int]:
        return [s.affected for s in self.series]


# ---------------------------------------------------------------- glue ---
def _device_landscape(land: Landscape, factor_site: str, slope_units: str,
                      wind=None) -> DeviceLandscape:
    if factor_site not in ("target", "source"):
        raise ValueError(f"factor_site must be 'target' or 'source', got {factor_site!r}")
    if slope_units not in ("degrees", "radians"):
        raise ValueError(f"slope_units must be 'degrees' or 'radians', got {slope_units!r}")
    vw = land.wind_speed if wind is None else wind[0]
    wd = land.wind_direction if wind is None else wind[1]
    return DeviceLandscape.from_slope_tensor(vw, wd, land.slope, land.canopy, land.density,
                                             cell_side=land.cell_side, factor_site=factor_site,
                                             slope_units=slope_units)


def _params8(params: ModelParams, norm_c: float):
    return pack_params(params.c1, params.c2, params.a, params.p_h, params.p_continue, norm_c)


def build_fields(land: Landscape, params: ModelParams, wind=None, *, with_gradients: bool = False,
                 norm_c: float = DEFAULT_NORM_C, factor_site: str = "target",
                 slope_units: str = "degrees") -> PropagationFields:
    """kernel.py:149-205: the eight per-slot probability fields (fp64, from
    the device).  The stencil itself never materialises them."""
    dl = _device_landscape(land, factor_site, slope_units, wind)
    out = build_fields_device(dl, _params8(params, norm_c), with_gradients).cpu().numpy()
    vw = np.asarray(wind[0] if wind else land.wind_speed, dtype=np.float64)
    f = PropagationFields(fp=out[:8], vw=vw, site_is_target=(factor_site == "target"))
    if with_gradients:
        f.raw, f.rest, f.cosm1, f.slope_toward = out[8:16], out[16:24], out[24:32], out[32:40]
    return f


def _pull_planes(batch: FireBatch, state: FireState):
    b, d = batch.unpack()
    state.burning[...] = b[0].bool().cpu().numpy()
    state.burned[...] = d[0].bool().cpu().numpy()


def _push_state(state: FireState, land_shape, max_steps) -> FireBatch:
    batch = FireBatch(land_shape, 1, max_steps=max_steps, record_live=True)
    batch.reset(state.burning, t0=state.t)
    if state.burned.any():
        _load_burned(batch, state)
    return batch


def _load_burned(batch: FireBatch, state: FireState):
    """Upload the burned cells of a host FireState into both burned planes."""
    h, w = batch.h, batch.w
    ty, tx = batch.grid.tiles_y, batch.grid.tiles_x
    burned = np.ones((ty * 32, tx * 32), dtype=bool)   # padding counts as burned
    burned[:h, :w] = state.burned
    bits = np.packbits(burned.reshape(ty, 32, tx, 32).transpose(0, 2, 1, 3), axis=-1,
                       bitorder="little").view(np.uint32).reshape(-1)
    batch.planes[2:4].copy_(torch.from_numpy(bits.view(np.int32)).expand(2, -1))
    batch.mark_cells_dirty()


def _check_fields(fields: PropagationFields, dl: DeviceLandscape, params8, factor_site: str):
    """step_forward(fields=...) (kernel.py:288-293): the device step derives
    the per-slot fields from the landscape in fp64 (fc_build_fields, the
    reference's operation order), so caller fields must be those fields --
    anything else is refused rather than silently replaced."""
    if fields.site_is_target != (factor_site == "target"):
        raise ValueError("fields were built for a different factor_site")
    want = build_fields_device(dl, params8, False).cpu().numpy()
    got = np.asarray(fields.fp, dtype=np.float64)
    h, w = dl.shape
    if got.shape != want.shape:
        raise ValueError(f"fields shape {got.shape} != {want.shape}")
    # targets off the grid are never consumed (kernel.py:117-125)
    inside = np.zeros((8, h, w), dtype=bool)
    for k, (pr, pc) in enumerate(NEIGHBOR_POSITIONS):
        inside[k, max(pr, 0):h + min(pr, 0), max(pc, 0):w + min(pc, 0)] = True
    if not np.allclose(got[inside], want[inside], rtol=1e-12, atol=0.0):
        raise ValueError("fields differ from build_fields(land, params): the device step "
                         "derives its per-slot fields from the landscape")


def step_forward(state: FireState, land: Landscape, params: ModelParams, seed: int, *,
                 attach: bool = False, tape: Optional[Tape] = None,
                 fields: Optional[PropagationFields] = None, threads: int = 1, executor=None,
                 norm_c: float = DEFAULT_NORM_C, factor_site: str = "target") -> FireState:
    """kernel.py:263-333: advance the state one step in place.  The step
    runs on the device; the ignitions' p_ignite (and J when attached) are
    recomputed in fp64 (fc_recompute64), so the host accumulator stays fp64
    like the reference's."""
    if state.shape != land.shape:
        raise ValueError(f"state shape {state.shape} != landscape {land.shape}")
    if attach and tape is None:
        raise ValueError("attach=True requires a tape")
    if attach and fields is not None and not fields.has_gradients:
        raise ValueError("attached step needs fields built with_gradients=True")
    dl = _device_landscape(land, factor_site, "degrees")
    p8 = _params8(params, norm_c)
    if fields is not None:
        _check_fields(fields, dl, p8, factor_site)
    t = state.t
    batch = _push_state(state, land.shape, t + 1)
    batch.set_params(p8)
    batch.set_seeds([seed])
    batch.run(dl, 1)
    acc64 = torch.as_tensor(np.asarray(state.accumulator, dtype=np.float64),
                            device=batch.device).reshape(1, *land.shape).contiguous()
    jac64 = (torch.zeros((1, *land.shape, 4), dtype=torch.float64, device=batch.device)
             if attach else None)
    batch.recompute64(dl, t, t + 1, acc64, jac64)
    _pull_planes(batch, state)
    state.accumulator[...] = acc64[0].cpu().numpy()
    if attach:
        n = int(batch.counters[0, t, 0].item())
        tape.bind(RunBinding(batch, jac64, acc64, [(t, t + 1, dl, p8, land.wind_speed)], [t + 1],
                             {t + 1: n}, norm_c, land.canopy, land.density,
                             factor_site == "target"))
    state.t = t + 1
    return state


def inject_ignitions(state: FireState, cells: Sequence[Tuple[int, int]]) -> FireState:
    """kernel.py:405-419 (host state; FireBatch.inject is the device form)."""
    h, w = state.shape
    for r, c in cells:
        if not (0 <= r < h and 0 <= c < w):
            raise IndexError(f"ignition cell ({r}, {c}) outside {h}x{w} grid")
        if state.burned[r, c] or state.burning[r, c]:
            continue
        state.burning[r, c] = True
        state.accumulator[r, c] = 1.0
    return state


def run_simulation(land: Landscape, params: ModelParams, init, steps: int, seed: int, *,
                   wind_schedule: Optional[Sequence[WindUpdate]] = None,
                   attach_steps: Iterable[int] = (), tape: Optional[Tape] = None,
                   snapshot_every: int = 0, threads: int = 1, norm_c: float = DEFAULT_NORM_C,
                   factor_site: str = "target", slope_units: str = "degrees",
                   rng: str = "splitmix", draws=None) -> SimulationResult:
    """kernel.py:453-529 on the device.  threads is accepted for signature
    compatibility (results are partition-invariant either way).  The
    accumulator (and the tape's Jacobians) are recomputed in fp64 from the
    run's live-slot masks (fc_recompute64), so results keep the reference's
    fp64 precision.  Extra keywords: rng ("splitmix" = the reference's
    draws, "philox", "inject") and draws ((steps, 2, H, W) fp64 uniforms for
    rng="inject")."""
    if steps < 0:
        raise ValueError("steps must be >= 0")
    schedule = sorted(wind_schedule or [], key=lambda u: u.apply_at_step)
    for upd in schedule:
        if not 1 <= upd.apply_at_step <= max(steps, 0):
            raise ValueError(f"wind schedule step {upd.apply_at_step} outside run of {steps} steps")
        if np.shape(upd.wind_speed) != land.shape or np.shape(upd.wind_direction) != land.shape:
            raise ValueError("scheduled wind field shape mismatch")
    attach_set = frozenset(int(s) for s in attach_steps)
    if attach_set and tape is None:
        tape = Tape(land.shape)
    state0 = new_fire_state(init, land)
    dl = _device_landscape(land, factor_site, slope_units)
    p8 = _params8(params, norm_c)
    batch = FireBatch(land.shape, 1, max_steps=max(steps, 1), record_live=True)
    batch.set_params(p8)
    batch.set_seeds([seed])
    batch.reset(state0.burning)
    if draws is not None:
        draws = torch.as_tensor(np.asarray(draws, dtype=np.float64)).reshape(steps, 1, 2, *land.shape)

    # segment boundaries: wind updates (applied before their 1-based step)
    # and snapshot points
    cuts = {1, steps + 1}
    cuts |= {u.apply_at_step for u in schedule}
    if snapshot_every:
        cuts |= {s + 1 for s in range(snapshot_every, steps + 1, snapshot_every)}
    # runs beyond the int16 ignition-step span rebase between segments
    span = FireBatch.REBASE_SPAN
    cuts |= set(range(span + 1, steps + 1, span))
    cuts = sorted(c for c in cuts if 1 <= c <= steps + 1)
    if attach_set and steps > span and min(attach_set) <= ((steps - 1) // span) * span:
        raise ValueError(f"attached steps must lie in the last {span} steps of a longer run")
    pending = list(schedule)
    vw_now = land.wind_speed
    segments = []      # (t_lo, t_hi, landscape, params8, wind speed) per run segment
    # p_ignite of every ignition (and J of the attached ones) in fp64, per
    # segment as it completes (fc_recompute64 from the live-slot masks)
    acc64 = torch.as_tensor(state0.accumulator, device=batch.device).reshape(1, *land.shape)
    acc64 = acc64.contiguous()
    jac64 = (torch.zeros((1, *land.shape, 4), dtype=torch.float64, device=batch.device)
             if attach_set else None)
    snapshots: List[Tuple[int, FireState]] = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        while pending and pending[0].apply_at_step == a:
            upd = pending.pop(0)
            dl = dl.with_wind(upd.wind_speed, upd.wind_direction)
            vw_now = upd.wind_speed
        if batch.t + (b - a) - batch.t_base > span:
            batch.rebase()
        seg_draws = None
        if draws is not None:
            seg_draws = draws[a - 1:b - 1]
        batch.run(dl, b - a, rng=rng, draws=seg_draws)
        batch.recompute64(dl, a - 1, b - 1, acc64, jac64)
        segments.append((a - 1, b - 1, dl, p8, vw_now))
        if snapshot_every and (b - 1) % snapshot_every == 0 and b - 1 >= 1:
            st = FireState(np.zeros(land.shape, bool), np.zeros(land.shape, bool),
                           acc64[0].cpu().numpy(), b - 1)
            _pull_planes(batch, st)
            snapshots.append((b - 1, st))
    final = FireState(np.zeros(land.shape, bool), np.zeros(land.shape, bool), np.zeros(land.shape),
                      steps)
    _pull_planes(batch, final)
    final.accumulator[...] = acc64[0].cpu().numpy()
    ser = batch.series()[0] if steps > 0 else np.zeros((0, 2), np.int64)
    series = [StepStats(t=i + 1, burning=int(ser[i, 0]), burned=int(ser[i, 1]))
              for i in range(steps)]
    if attach_set:
        cnt = batch.counters[0, :max(steps, 1), 0].cpu().numpy()
        steps_in = sorted(s for s in attach_set if 1 <= s <= steps)
        tape.bind(RunBinding(batch, jac64, acc64, segments, steps_in,
                             {s: int(cnt[s - 1]) for s in steps_in}, norm_c, land.canopy,
                             land.density, factor_site == "target"))
    res = SimulationResult(state=final, series=series, snapshots=snapshots, tape=tape)
    res.batch = batch  # device state (t_ign, live masks)
    return res
