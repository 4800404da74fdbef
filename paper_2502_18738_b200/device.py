"""Device-resident landscape and fire state (the native B200 API).

``DeviceLandscape`` holds the HBM layout of one landscape; ``FireBatch``
holds M independent fire states sharing it (an ensemble; M = 1 for the
reference's single-simulation API) and drives the kernels of
libfirecell.so through the C ABI (include/firecell.h).  PyTorch provides
device memory and streams only.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as L

# Slot order NW,N,NE,W,E,SW,S,SE (pyrocell/kernel.py:30-34)
NEIGHBOR_POSITIONS = ((-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1))
DEFAULT_NORM_C = 1.1486328125


def _u64_to_i64(v: int) -> int:
    v = int(v) & (2**64 - 1)
    return v - 2**64 if v >= 2**63 else v


def _dev(device) -> torch.device:
    d = torch.device(device if device is not None else "cuda")
    if d.type != "cuda":
        raise RuntimeError("firecell runs on CUDA devices only (no CPU fallback)")
    return d


def _build_from_rasters(rasters, cell_side: float, sign: int, dev):
    """fc_landscape_build: (env, slope4, env64, dir32) from five same-shape
    rasters (elevation, wind speed, wind direction, canopy, density), fp32 or
    fp64, in one device pass (fp64 arithmetic, the reference's preparation
    order, data_io.py:92-132 and model.py:76-105)."""
    ts = [torch.as_tensor(np.asarray(a) if not torch.is_tensor(a) else a) for a in rasters]
    shape = tuple(ts[0].shape)
    if len(shape) != 2 or any(tuple(t.shape) != shape for t in ts):
        raise ValueError("landscape rasters must be 2-D and of one shape")
    # fp32 rasters stay fp32 (widened exactly in the kernel); anything else
    # is taken in fp64
    dt = torch.float32 if all(t.dtype == torch.float32 for t in ts) else torch.float64
    ts = [t.to(dev, dt).contiguous() for t in ts]
    h, w = shape
    env = torch.empty((h, w, 4), dtype=torch.float32, device=dev)
    slope4 = torch.empty((h, w, 4), dtype=torch.float32, device=dev)
    env64 = torch.empty((h, w, 5), dtype=torch.float64, device=dev)
    dir32 = torch.empty((h, w, 2), dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        L.check(L.lib().fc_landscape_build(
            h, w, *[L.ptr(t) for t in ts], 1 if dt == torch.float64 else 0, float(cell_side),
            -1 if sign < 0 else 1, L.ptr(env), L.ptr(slope4), L.ptr(env64), L.ptr(dir32),
            L.stream_ptr()), "fc_landscape_build")
    return env, slope4, env64, dir32


class DeviceLandscape:
    """Environment rasters in the kernel's layout (see include/firecell.h).

    env fp32 [H][W][4] = (elevation, wind east, wind north, vd) feeds the
    fp32 fast path; env64 fp64 [H][W][5] = (elevation, speed, direction,
    canopy, density) feeds the rare fp64 guard recompute; the optional slope
    tensors [H][W][8] replace the elevation-derived slope.
    """

    def __init__(self, env: torch.Tensor, env64: torch.Tensor, *, cell_side: float = 30.0,
                 slope32: Optional[torch.Tensor] = None, slope64: Optional[torch.Tensor] = None,
                 slope_sign: int = 1, factor_site: str = "target",
                 slope4: Optional[torch.Tensor] = None, dir32: Optional[torch.Tensor] = None):
        if factor_site not in ("target", "source"):
            raise ValueError(f"factor_site must be 'target' or 'source', got {factor_site!r}")
        self.env, self.env64 = env.contiguous(), env64.contiguous()
        if slope4 is None or dir32 is None:
            # derived planes from the fp64 rasters (fc_landscape_build)
            _, s4, _, d32 = _build_from_rasters([self.env64[..., i] for i in range(5)],
                                                cell_side, slope_sign, self.env64.device)
            slope4 = s4 if slope4 is None else slope4
            dir32 = d32 if dir32 is None else dir32
        self.slope4 = slope4
        self.dir32 = dir32.contiguous()
        self.slope32 = None if slope32 is None else slope32.contiguous()
        self.slope64 = None if slope64 is None else slope64.contiguous()
        self.cell_side = float(cell_side)
        self.slope_sign = -1 if slope_sign < 0 else 1
        self.factor_site = factor_site
        self.shape = tuple(env.shape[:2])

    # ---------------------------------------------------------- builders
    @classmethod
    def from_elevation(cls, elevation, wind_speed, wind_direction, canopy, density, *,
                       cell_side: float = 30.0, slope_sign: str = "downhill-positive",
                       factor_site: str = "target", device=None) -> "DeviceLandscape":
        """Elevation mode: slope derived on the fly per live pair (the fused
        slope_from_altitude, pyrocell/data_io.py:92-132)."""
        dev = _dev(device)
        if slope_sign not in ("downhill-positive", "uphill-positive"):
            raise ValueError(f"unknown slope_sign {slope_sign!r}")
        if cell_side <= 0:
            raise ValueError("cell_side must be > 0")
        sign = -1 if slope_sign == "uphill-positive" else 1
        env, slope4, env64, dir32 = _build_from_rasters(
            (elevation, wind_speed, wind_direction, canopy, density), cell_side, sign, dev)
        return cls(env, env64, cell_side=cell_side, slope_sign=sign, factor_site=factor_site,
                   slope4=slope4, dir32=dir32)

    @classmethod
    def from_environment(cls, env, **kw) -> "DeviceLandscape":
        return cls.from_elevation(env.elevation, env.wind_speed, env.wind_direction, env.canopy,
                                  env.density, cell_side=env.cell_side, **kw)

    @classmethod
    def from_slope_tensor(cls, wind_speed, wind_direction, slope, canopy, density, *,
                          cell_side: float = 30.0, factor_site: str = "target",
                          slope_units: str = "degrees", device=None) -> "DeviceLandscape":
        """Slope-tensor mode for the reference Landscape (model.py:76-105):
        slope (H, W, 3, 3) degrees from each cell toward each neighbour."""
        dev = _dev(device)
        if slope_units not in ("degrees", "radians"):
            raise ValueError(f"slope_units must be 'degrees' or 'radians', got {slope_units!r}")
        sl = np.asarray(slope, dtype=np.float64)
        if slope_units == "radians":
            sl = np.degrees(sl)
        h, w = sl.shape[:2]
        # slot k at the source: slope toward the target = source - position
        s8 = np.stack([sl[:, :, 1 - pr, 1 - pc] for pr, pc in NEIGHBOR_POSITIONS], axis=-1)
        zeros = np.zeros((h, w))
        base = cls.from_elevation(zeros, wind_speed, wind_direction, canopy, density,
                                  cell_side=cell_side, factor_site=factor_site, device=dev)
        s64 = torch.as_tensor(np.ascontiguousarray(s8)).to(dev)
        base.slope64 = s64
        base.slope32 = s64.to(torch.float32)
        return base

    def with_wind(self, wind_speed, wind_direction) -> "DeviceLandscape":
        """Same landscape with replaced wind fields (WindUpdate, kernel.py:422-428),
        rebuilt by fc_landscape_build (the elevation-derived slope is kept)."""
        e64 = self.env64
        env, _, env64, dir32 = _build_from_rasters(
            (e64[..., 0], wind_speed, wind_direction, e64[..., 3], e64[..., 4]), self.cell_side,
            self.slope_sign, self.env.device)
        return DeviceLandscape(env, env64, cell_side=self.cell_side, slope32=self.slope32,
                               slope64=self.slope64, slope_sign=self.slope_sign,
                               factor_site=self.factor_site, slope4=self.slope4, dir32=dir32)

    def struct(self) -> L.FcLandscape:
        s = L.FcLandscape()
        s.env, s.env64 = L.ptr(self.env), L.ptr(self.env64)
        s.slope4 = L.ptr(self.slope4)
        s.slope32, s.slope64 = L.ptr(self.slope32), L.ptr(self.slope64)
        s.dir32 = L.ptr(self.dir32)
        s.cell_side = self.cell_side
        s.slope_mode = L.SLOPE_TENSOR if self.slope64 is not None else L.SLOPE_ELEVATION
        s.slope_sign = self.slope_sign
        s.factor_source = 1 if self.factor_site == "source" else 0
        return s

    @property
    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in
                   (self.env, self.slope4, self.env64, self.dir32, self.slope32, self.slope64)
                   if t is not None)


def wind_ramp_schedule(steps: int, v_start: float = 2.0, v_end: float = 12.0,
                       rotate_deg: float = 90.0, keep_field: bool = False,
                       device=None) -> torch.Tensor:
    """Per-step wind schedule of BASELINE config 4: the direction rotates
    linearly by rotate_deg over the run and the speed ramps linearly from
    v_start to v_end (uniform speed; keep_field=True scales the base field
    instead).  Row t = {alpha, beta, gamma_deg, 0} for pre-step index t."""
    frac = np.arange(steps, dtype=np.float64) / max(steps - 1, 1)
    speed = v_start + (v_end - v_start) * frac
    sched = np.zeros((steps, 4), dtype=np.float64)
    if keep_field:
        sched[:, 0] = speed / max(v_start, 1e-12)
    else:
        sched[:, 1] = speed
    sched[:, 2] = rotate_deg * frac
    return torch.as_tensor(sched, device=device if device is not None else "cuda")


def scheduled_wind_fields(speed, direction, row):
    """fp64 host fields one schedule row implies (for the reference API /
    oracle): speed' = alpha * speed + beta, direction' = direction + gamma."""
    a, b, g = float(row[0]), float(row[1]), float(row[2])
    return a * np.asarray(speed, dtype=np.float64) + b, np.asarray(direction, dtype=np.float64) + g


def pack_params(c1, c2, a, p_h, p_continue, norm_c=DEFAULT_NORM_C) -> list:
    return [float(c1), float(c2), float(a), float(p_h), float(p_continue), float(norm_c), 0.0, 0.0]


class FireBatch:
    """M fire states on one landscape: bit planes, accumulator, ignition
    steps, per-cell Jacobians, activity flags and per-step counters."""

    def __init__(self, shape, members: int = 1, *, max_steps: int = 1024,
                 with_jacobian: bool = False, member0: int = 0, record_live: bool = False,
                 dataflow: bool = True, device=None):
        """member0: global index of local member 0 when an ensemble is
        sharded over ranks (the member word of the Philox counter).
        record_live: keep each ignition's live-slot mask (1 B per cell), which
        recompute64() turns into fp64 accumulators and Jacobians.
        dataflow: ensembles (members >= 2) run each run() call as one
        persistent launch in which members advance independently
        (fc_state.sched); False keeps one launch per window."""
        L.require_cuda()
        dev = _dev(device)
        self.device = dev
        if member0 < 0:
            raise ValueError("member0 must be >= 0")
        self.member0 = int(member0)
        self.h, self.w = int(shape[0]), int(shape[1])
        if self.h < 1 or self.w < 1:
            raise ValueError(f"grid must be at least 1x1, got {shape}")
        self.m = int(members)
        self.grid = L.grid(self.h, self.w, self.m)
        words = L.lib().fc_plane_words(C.byref(self.grid))
        self.planes = torch.empty((4, words), dtype=torch.int32, device=dev)
        hw = self.h * self.w
        self.acc = torch.zeros((self.m, self.h, self.w), dtype=torch.float32, device=dev)
        self.t_ign = torch.empty((self.m, self.h, self.w), dtype=torch.int16, device=dev)
        self.jac = (torch.zeros((self.m, self.h, self.w, 4), dtype=torch.float32, device=dev)
                    if with_jacobian else None)
        self.live = (torch.zeros((self.m, self.h, self.w), dtype=torch.uint8, device=dev)
                     if record_live else None)
        self.flags = torch.empty((self.m, self.grid.tiles_y, self.grid.tiles_x), dtype=torch.int32,
                                 device=dev)
        self.max_steps = int(max_steps)
        self.counters = torch.zeros((self.m, self.max_steps, L.NCOUNTER), dtype=torch.int32,
                                    device=dev)
        # launches are bounded by steps (>= 1 step per launch) plus resets' lists
        ntiles = self.m * self.grid.tiles_y * self.grid.tiles_x
        self.tile_list = torch.empty((3, ntiles), dtype=torch.int32, device=dev)
        self.list_count = torch.zeros((2 * (self.max_steps + 3) + 4,), dtype=torch.int32, device=dev)
        self.tile_fire = torch.zeros((ntiles,), dtype=torch.uint8, device=dev)
        self.tile_first = torch.full((ntiles,), L.T_NEVER, dtype=torch.int32, device=dev)
        self._cells_clean = False  # acc / t_ign hold no library-written state yet
        self._mode = None  # sweep mode since reset (activity lists vs dense rescans)
        self.params = torch.zeros((self.m, L.NPARAM), dtype=torch.float64, device=dev)
        self.seeds = torch.zeros((self.m,), dtype=torch.int64, device=dev)
        self.adam = torch.zeros((self.m, 8), dtype=torch.float64, device=dev)
        self.adam_step = torch.zeros((self.m,), dtype=torch.int32, device=dev)
        self._status = torch.zeros((self.m,), dtype=torch.int32, device=dev)
        ws = max(L.lib().fc_loss_workspace_bytes(C.byref(self.grid), 8), 1 << 12)
        self.workspace = torch.empty((ws,), dtype=torch.uint8, device=dev)
        # ensembles: the dataflow scheduler's workspace (fc_state.sched)
        self.sched = (torch.empty((L.lib().fc_sched_workspace_bytes(C.byref(self.grid),
                                                                    self.max_steps),),
                                  dtype=torch.uint8, device=dev)
                      if self.m >= 2 and dataflow else None)
        self.t = 0
        self.t_base = 0  # t_ign / tile_first count steps from here (fc_state.t_base)
        self.q = 0  # launches since reset (burning-buffer parity, activity lists)
        self._init_burning_dev = torch.zeros((self.m,), dtype=torch.int64, device=dev)
        self._hw = hw

    @property
    def init_burning(self) -> np.ndarray:
        """Burning cells per member at the last reset (host copy on demand)."""
        return self._init_burning_dev.cpu().numpy().copy()

    # ------------------------------------------------------------ plumbing
    def struct(self) -> L.FcState:
        # the state's buffers never move: build the descriptor once
        if getattr(self, "_struct", None) is not None:
            return self._struct
        s = L.FcState()
        base, stride = self.planes.data_ptr(), self.planes.stride(0) * 4
        s.burn0, s.burn1 = base, base + stride
        s.burned0, s.burned1 = base + 2 * stride, base + 3 * stride
        s.acc, s.t_ign, s.jac = L.ptr(self.acc), L.ptr(self.t_ign), L.ptr(self.jac)
        s.flags, s.counters = L.ptr(self.flags), L.ptr(self.counters)
        s.tile_list, s.list_count = L.ptr(self.tile_list), L.ptr(self.list_count)
        s.tile_fire = L.ptr(self.tile_fire)
        s.tile_first = L.ptr(self.tile_first)
        s.live = L.ptr(self.live)
        s.sched = L.ptr(self.sched)
        s.init_burning = L.ptr(self._init_burning_dev)
        s.max_steps = self.max_steps
        s.t_base = self.t_base
        self._struct = s
        return s

    def set_params(self, params: Sequence, member: Optional[int] = None):
        """params: 8-vectors (see pack_params) for every member or one."""
        p = torch.as_tensor(np.asarray(params, dtype=np.float64), device=self.device)
        if member is None:
            self.params.copy_(p.reshape(-1, L.NPARAM).expand(self.m, L.NPARAM))
        else:
            self.params[member].copy_(p.reshape(L.NPARAM))

    def set_seeds(self, seeds):
        s = [_u64_to_i64(v) for v in np.atleast_1d(np.asarray(seeds, dtype=object))]
        if len(s) == 1:
            s = s * self.m
        self.seeds.copy_(torch.tensor(s, dtype=torch.int64))

    # -------------------------------------------------------------- state
    def reset(self, init, t0: int = 0, stream=None):
        """new_fire_state (model.py:180-200) for every member; init is a
        (H, W) mask broadcast to all members or an (M, H, W) stack."""
        if torch.is_tensor(init):
            m8 = init.to(self.device, torch.uint8)
        else:
            m8 = torch.as_tensor(np.asarray(init, dtype=bool).astype(np.uint8), device=self.device)
        if m8.dim() == 2:
            if tuple(m8.shape) != (self.h, self.w):
                raise ValueError(f"initial fire mask shape {tuple(m8.shape)} != landscape {(self.h, self.w)}")
            stride = 0
        elif m8.dim() == 3 and tuple(m8.shape) == (self.m, self.h, self.w):
            stride = self._hw
        else:
            raise ValueError(f"initial fire mask must be 2-D or (M,H,W), got {tuple(m8.shape)}")
        # the reset kernels count the initial burning cells into
        # _init_burning_dev (fc_state.init_burning): no host sync inside a
        # timed or captured sequence; series() reads them when asked
        self._init_mask = m8.contiguous()
        st = self.struct()
        # after the first full initialisation only the tiles that held fire
        # are rewritten (fc_state_reset); external writes to acc / t_ign
        # must call mark_cells_dirty() first
        fn = L.lib().fc_state_reset if self._cells_clean else L.lib().fc_state_init
        L.check(fn(C.byref(self.grid), C.byref(st), L.ptr(self._init_mask), stride, int(t0),
                   L.stream_ptr(stream)), "fc_state_init")
        self._cells_clean = True
        self.t = int(t0)
        self._set_base(int(t0))
        self.q = 0
        self._mode = None

    # --------------------------------------------------------- long runs
    REBASE_SPAN = 30000  # steps between bases (int16 t_ign spans 32766)

    def _set_base(self, t_base: int):
        self.t_base = int(t_base)
        if getattr(self, "_struct", None) is not None:
            self._struct.t_base = self.t_base

    def rebase(self, stream=None):
        """fc_state_rebase: ignitions recorded so far count as "before the
        base" (t_ign -1) and the base moves to the current step, so runs may
        exceed the int16 ignition-step range (kernel.py:453-468 has no step
        limit).  Losses, tape steps and recompute64 then address ignitions
        after this point only."""
        st = self.struct()
        L.check(L.lib().fc_state_rebase(C.byref(self.grid), C.byref(st), L.stream_ptr(stream)),
                "fc_state_rebase")
        self._set_base(self.t)

    def run(self, land: DeviceLandscape, nsteps: int, *, attach: Optional[Sequence[bool]] = None,
            rng: str = "splitmix", draws: Optional[torch.Tensor] = None, skip_inactive: bool = True,
            window: Optional[int] = None, wind_schedule: Optional[torch.Tensor] = None, shard=None,
            stream=None):
        """Advance every member nsteps steps from the current pre-step index,
        `window` steps per kernel launch (temporal blocking; 1, 4, 8, 16;
        default 16 for one or two members, else 8).
        wind_schedule: optional fp64 (max_steps, 4) device tensor of per-step
        {alpha, beta, gamma_deg, 0} (see wind_ramp_schedule)."""
        if nsteps < 0:
            raise ValueError("steps must be >= 0")
        if land.shape != (self.h, self.w):
            raise ValueError(f"state shape {(self.h, self.w)} != landscape {land.shape}")
        if self.t + nsteps > self.max_steps:
            raise ValueError(f"run past max_steps={self.max_steps}")
        if self.t + nsteps - self.t_base > self.REBASE_SPAN:
            # beyond the int16 ignition-step range: advance in spans, moving
            # the base forward between them (the launch parity carries over)
            while nsteps > 0:
                room = self.t_base + self.REBASE_SPAN - self.t
                if room <= 0:
                    self.rebase(stream)
                    continue
                n = min(nsteps, room)
                self.run(land, n, attach=None if attach is None else list(attach)[:n], rng=rng,
                         draws=None if draws is None else draws[:n],
                         skip_inactive=skip_inactive, window=window,
                         wind_schedule=wind_schedule, shard=shard, stream=stream)
                attach = None if attach is None else list(attach)[n:]
                draws = None if draws is None else draws[n:]
                nsteps -= n
            return
        att = None
        if attach is not None:
            att_np = np.ascontiguousarray(np.asarray(attach, dtype=np.uint8)[:nsteps])
            if att_np.any() and self.jac is None:
                raise ValueError("attached steps need a FireBatch built with_jacobian=True")
            att = att_np.ctypes.data_as(C.c_void_p)
        mode = L.RNG_MODES[rng]
        if mode == L.RNG_INJECT:
            if draws is None or tuple(draws.shape) != (nsteps, self.m, 2, self.h, self.w):
                raise ValueError("inject mode needs draws of shape (nsteps, M, 2, H, W)")
            draws = draws.to(self.device, torch.float64).contiguous()
        if window is None:
            # one or two members are latency-bound: longer windows halve the
            # launches; ensembles are throughput-bound: shorter halos, and
            # the shortest for the largest (attached c4 shape, 1024^2 x 200
            # steps: K=8 faster up to 128 members, K=4 at 256: 3.50 vs 3.61 ms)
            window = 16 if self.m <= 2 else (4 if self.m >= 256 else 8)
        if window not in (1, 4, 8, 16):
            raise ValueError("window must be 1, 4, 8 or 16")
        if self._mode is not None and self._mode != bool(skip_inactive):
            raise ValueError("skip_inactive cannot change between runs without reset()")
        self._mode = bool(skip_inactive)
        if wind_schedule is not None:
            if tuple(wind_schedule.shape) != (self.max_steps, 4) or wind_schedule.dtype != torch.float64:
                raise ValueError("wind_schedule must be fp64 of shape (max_steps, 4)")
            wind_schedule = wind_schedule.to(self.device).contiguous()
        lst, st = land.struct(), self.struct()
        if shard is None and self.member0:
            shard = L.FcShard(0, 0, 0, self.member0)
        elif shard is not None:
            shard.member0 = self.member0
        phase = C.c_int32(self.q)
        L.check(L.lib().fc_run(C.byref(self.grid), C.byref(lst), C.byref(st), L.ptr(self.params),
                               L.ptr(self.seeds), mode, L.ptr(draws), self.t, int(nsteps), att,
                               1 if skip_inactive else 0, int(window), L.ptr(wind_schedule),
                               None if shard is None else C.byref(shard), C.byref(phase),
                               L.stream_ptr(stream)), "fc_run")
        self.t += int(nsteps)
        self.q = int(phase.value)
        self._keep = (att_np if attach is not None else None, draws)  # lifetime until sync

    def run_pass(self, land: DeviceLandscape, nsteps: int, window: int, which: int, shard,
                 *, attach: Optional[Sequence[bool]] = None, rng: str = "splitmix",
                 wind_schedule: Optional[torch.Tensor] = None, stream=None):
        """One window launch of a row shard in two passes (fc_run_pass):
        which = 1 advances the listed tiles away from the ghost rows (the
        step index and launch phase stay), which = 2 the boundary tile rows
        (then both advance).  Same bytes as run() on the whole launch."""
        if which not in (1, 2):
            raise ValueError("which must be 1 (interior) or 2 (boundary rows)")
        if not 1 <= nsteps <= window or window not in (1, 4, 8, 16):
            raise ValueError("a pass covers one launch of 1..window steps")
        if self.t + nsteps > self.max_steps:
            raise ValueError(f"run past max_steps={self.max_steps}")
        if self._mode is False:
            raise ValueError("split launches need activity lists (skip_inactive=True)")
        self._mode = True
        att = None
        if attach is not None:
            att_np = np.ascontiguousarray(np.asarray(attach, dtype=np.uint8)[:nsteps])
            if att_np.any() and self.jac is None:
                raise ValueError("attached steps need a FireBatch built with_jacobian=True")
            att = att_np.ctypes.data_as(C.c_void_p)
        if wind_schedule is not None:
            if tuple(wind_schedule.shape) != (self.max_steps, 4) or wind_schedule.dtype != torch.float64:
                raise ValueError("wind_schedule must be fp64 of shape (max_steps, 4)")
        shard.member0 = self.member0
        lst, st = land.struct(), self.struct()
        phase = C.c_int32(self.q)
        L.check(L.lib().fc_run_pass(C.byref(self.grid), C.byref(lst), C.byref(st),
                                    L.ptr(self.params), L.ptr(self.seeds), L.RNG_MODES[rng],
                                    self.t, int(nsteps), att, int(window), L.ptr(wind_schedule),
                                    C.byref(shard), int(which), C.byref(phase),
                                    L.stream_ptr(stream)), "fc_run_pass")
        if which == 2:
            self.t += int(nsteps)
            self.q = int(phase.value)

    def inject(self, cells, member: int = 0, stream=None):
        """inject_ignitions (kernel.py:405-419) before the current step."""
        rows = []
        for cell in cells:
            if len(cell) == 3:
                m, r, c = (int(v) for v in cell)
            else:
                m, (r, c) = member, (int(cell[0]), int(cell[1]))
            if not (0 <= r < self.h and 0 <= c < self.w):
                raise IndexError(f"ignition cell ({r}, {c}) outside {self.h}x{self.w} grid")
            rows.append((m, r, c))
        if not rows:
            return
        t = torch.tensor(rows, dtype=torch.int32, device=self.device)
        st = self.struct()
        L.check(L.lib().fc_inject(C.byref(self.grid), C.byref(st), L.ptr(t), len(rows), self.t,
                                  self.q, L.stream_ptr(stream)), "fc_inject")
        self._inj = t

    def mark_cells_dirty(self):
        """Call after writing acc or t_ign directly: the next reset then
        rewrites every cell instead of only the tiles that held fire."""
        self._cells_clean = False

    def unpack(self, stream=None):
        """(burning, burned) uint8 tensors (M, H, W) at the current step."""
        b = torch.empty((self.m, self.h, self.w), dtype=torch.uint8, device=self.device)
        d = torch.empty_like(b)
        st = self.struct()
        L.check(L.lib().fc_state_unpack(C.byref(self.grid), C.byref(st), self.q, L.ptr(b),
                                        L.ptr(d), L.stream_ptr(stream)), "fc_state_unpack")
        return b, d

    def jaccard(self, targets: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None):
        """fc_state_jaccard: per-member Jaccard index (losses.py:89-98) of the
        affected cells (burning | burned) against uint8/bool targets (H, W)
        shared by all members, or (M, H, W); from the bit planes, on the
        device.  Returns a float64 (M,) device tensor (out, if given)."""
        t = targets if targets.dtype == torch.uint8 else targets.to(torch.uint8)
        t = t.to(self.device).contiguous()
        if t.shape[-2:] != (self.h, self.w) or (t.dim() == 3 and t.shape[0] not in (1, self.m)):
            raise ValueError(f"targets shape {tuple(t.shape)} does not match {(self.m, self.h, self.w)}")
        stride = self.h * self.w if t.dim() == 3 and t.shape[0] == self.m and self.m > 1 else 0
        if out is None:
            out = torch.empty((self.m,), dtype=torch.float64, device=self.device)
        if getattr(self, "_jaccard_work", None) is None:
            self._jaccard_work = torch.zeros((2 * self.m + 1,), dtype=torch.int64, device=self.device)
        st = self.struct()
        L.check(L.lib().fc_state_jaccard(C.byref(self.grid), C.byref(st), self.q, L.ptr(t), stride,
                                         L.ptr(self._jaccard_work), L.ptr(out),
                                         L.stream_ptr(stream)), "fc_state_jaccard")
        return out

    def export(self, burning, burned, acc, written=None, stream=None):
        """fc_state_export: the current state into (M, H, W) uint8 / uint8 /
        fp32 tensors (any may be None), on the device or pinned on the host
        (written by the kernel over PCIe).  written: None, or a uint8
        (M, TY, TX) device tensor of per-tile flags kept with a reused
        destination (zero-initialised with it): only affected tiles and
        tiles written last time are then touched."""
        for t, dt in ((burning, torch.uint8), (burned, torch.uint8), (acc, torch.float32)):
            if t is not None and (t.dtype != dt or tuple(t.shape) != (self.m, self.h, self.w)
                                  or not t.is_contiguous()):
                raise ValueError("export destinations must be contiguous (M, H, W) "
                                 "uint8 / uint8 / float32")
        if written is not None and (written.dtype != torch.uint8 or not written.is_cuda or
                                    written.numel() != self.m * self.grid.tiles_y * self.grid.tiles_x):
            raise ValueError("written must be a uint8 (M, TY, TX) device tensor")
        st = self.struct()
        L.check(L.lib().fc_state_export(C.byref(self.grid), C.byref(st), self.q,
                                        L.device_ptr(burning), L.device_ptr(burned),
                                        L.device_ptr(acc), L.ptr(written), L.stream_ptr(stream)),
                "fc_state_export")

    def series(self, t0: int = 0, t1: Optional[int] = None) -> np.ndarray:
        """Per-step (burning, burned) counts after each step in [t0, t1)
        (StepStats, kernel.py:431-439), from the device counters."""
        t1 = self.t if t1 is None else t1
        cnt = self.counters[:, :t1].to(torch.int64).cpu().numpy()
        burning = self.init_burning[:, None] + np.cumsum(cnt[:, :, 0] - cnt[:, :, 1], axis=1)
        burned = np.cumsum(cnt[:, :, 1], axis=1)
        return np.stack([burning, burned], axis=-1)[:, t0:t1]

    def attached_entries(self, attach_mask) -> int:
        """Number of tape entries: ignitions on attached steps."""
        cnt = self.counters[:, : self.t, 0].to(torch.int64).cpu().numpy()
        mask = np.zeros(self.t, dtype=bool)
        am = np.asarray(attach_mask, dtype=bool)
        mask[: min(len(am), self.t)] = am[: self.t]
        return int(cnt[:, mask].sum())

    # ------------------------------------------------------- fp64 outputs
    def recompute64(self, land: DeviceLandscape, t_lo: int, t_hi: int, acc64: torch.Tensor,
                    jac64: Optional[torch.Tensor] = None, wind_schedule=None, stream=None):
        """fc_recompute64: p_ignite (and J) in fp64 for the cells that ignited
        at pre-step indices [t_lo, t_hi) of this run, which ran on `land`;
        written into acc64 (M, H, W) / jac64 (M, H, W, 4) fp64 device tensors."""
        if self.live is None:
            raise ValueError("recompute64 needs a FireBatch built with record_live=True")
        for t, shp in ((acc64, (self.m, self.h, self.w)), (jac64, (self.m, self.h, self.w, 4))):
            if t is not None and (t.dtype != torch.float64 or tuple(t.shape) != shp or
                                  not t.is_contiguous() or not t.is_cuda):
                raise ValueError(f"expected a contiguous fp64 {shp} CUDA tensor")
        st = self.struct()
        L.check(L.lib().fc_recompute64(C.byref(self.grid), C.byref(land.struct()), C.byref(st),
                                       L.ptr(self.params), int(t_lo), int(t_hi),
                                       L.ptr(wind_schedule), L.ptr(acc64), L.ptr(jac64),
                                       L.stream_ptr(stream)), "fc_recompute64")

    def contract_steps(self, dl_dacc: torch.Tensor, jac64: torch.Tensor, steps,
                       stream=None) -> torch.Tensor:
        """backward_params over the ignitions of the given pre-step indices
        (tape blocks): (M, 4) = sum dL/dacc * J64 (fc_contract_steps)."""
        g = dl_dacc.to(self.device, torch.float64).reshape(self.m, self.h, self.w).contiguous()
        flags = torch.zeros((max(self.max_steps, 1),), dtype=torch.uint8)
        for t in steps:
            if 0 <= int(t) < flags.numel():
                flags[int(t)] = 1
        flags = flags.to(self.device)
        out = torch.empty((self.m, 4), dtype=torch.float64, device=self.device)
        st = self.struct()
        L.check(L.lib().fc_contract_steps(C.byref(self.grid), C.byref(st), L.ptr(g), L.ptr(jac64),
                                          L.ptr(flags), flags.numel(), L.ptr(out),
                                          L.ptr(self.workspace), L.stream_ptr(stream)),
                "fc_contract_steps")
        self._keep_c = (g, flags)
        return out

    # ----------------------------------------------------------- backward
    def contract(self, dl_dacc: torch.Tensor, stream=None) -> torch.Tensor:
        """backward_params (tape.py:118-148): (M, 4) = sum_j dL/dacc_j J_j."""
        if self.jac is None:
            raise ValueError("no Jacobian recorded (FireBatch(with_jacobian=False))")
        g = dl_dacc.to(self.device)
        if g.dtype not in (torch.float32, torch.float64):
            g = g.to(torch.float64)
        g = g.reshape(self.m, self.h, self.w).contiguous()
        out = torch.empty((self.m, 4), dtype=torch.float64, device=self.device)
        st = self.struct()
        L.check(L.lib().fc_contract(C.byref(self.grid), C.byref(st), L.ptr(g),
                                    1 if g.dtype == torch.float32 else 0, L.ptr(out),
                                    L.ptr(self.workspace), L.stream_ptr(stream)), "fc_contract")
        self._keep_g = g
        return out

    def loss_grad(self, targets: torch.Tensor, obs_steps: Sequence[int], *, per_member=False,
                  want_grad=True, want_dl_dacc=False, stream=None):
        """combined_loss summed over observation steps, fused with the
        gradient contraction.  targets: (S, H, W) shared or (S, M, H, W)."""
        S = len(obs_steps)
        tg = targets.to(self.device, torch.uint8).contiguous()
        if tg.dim() == 2:
            tg = tg[None]
        if tg.shape[0] != S:
            raise ValueError("one target per observation step")
        if tg.dim() == 3:
            if tuple(tg.shape[1:]) != (self.h, self.w):
                raise ValueError(f"target shape {tuple(tg.shape[1:])} != accumulator {(self.h, self.w)}")
            mstride = 0
        else:
            mstride = self._hw
        if any(int(s) < self.t_base for s in obs_steps):
            raise ValueError(f"observation steps before the last rebase (t_base={self.t_base})")
        obs = (C.c_int32 * S)(*[int(s) for s in obs_steps])
        loss = torch.empty((self.m, 2 + 2 * S), dtype=torch.float64, device=self.device)
        crop = torch.empty((self.m, S, 4), dtype=torch.int32, device=self.device)
        grad = torch.empty((self.m, 4), dtype=torch.float64, device=self.device) if want_grad else None
        dl = (torch.empty((self.m, self.h, self.w), dtype=torch.float64, device=self.device)
              if want_dl_dacc else None)
        st = self.struct()
        L.check(L.lib().fc_loss_grad(C.byref(self.grid), C.byref(st), L.ptr(tg), mstride, obs, S,
                                     L.ptr(loss), L.ptr(crop), L.ptr(grad), L.ptr(dl),
                                     L.ptr(self.workspace), L.stream_ptr(stream)), "fc_loss_grad")
        self._keep_t = tg
        return loss, crop, grad, dl

    def adamw(self, grads: torch.Tensor, step: Optional[int], lr: float, weight_decay: float = 0.0,
              beta1=0.9, beta2=0.999, eps=1e-8, clamp=True, stream=None) -> torch.Tensor:
        """AdamW + clamp on the device params; step=None uses the device step
        counter (self.adam_step), which keeps CUDA-graph replays valid."""
        status = self._status
        L.check(L.lib().fc_adamw(L.ptr(grads), L.ptr(self.params), L.ptr(self.adam), self.m,
                                 0 if step is None else int(step),
                                 L.ptr(self.adam_step) if step is None else None, lr,
                                 weight_decay, beta1, beta2, eps, 1 if clamp else 0,
                                 L.ptr(status), L.stream_ptr(stream)), "fc_adamw")
        return status


def loss_dense(acc: torch.Tensor, target: torch.Tensor, want_grad=True, stream=None):
    """combined_loss (losses.py:44-86) of an arbitrary fp64 accumulator."""
    L.require_cuda()
    a = acc.to("cuda", torch.float64).contiguous()
    y = target.to("cuda", torch.uint8).contiguous()
    h, w = a.shape
    g = L.grid(h, w, 1)
    ws = torch.empty((max(L.lib().fc_loss_workspace_bytes(C.byref(g), 1), 4096),),
                     dtype=torch.uint8, device=a.device)
    loss = torch.empty((4,), dtype=torch.float64, device=a.device)
    crop = torch.empty((4,), dtype=torch.int32, device=a.device)
    dl = torch.empty_like(a) if want_grad else None
    L.check(L.lib().fc_loss_dense(h, w, L.ptr(a), L.ptr(y), L.ptr(loss), L.ptr(crop), L.ptr(dl),
                                  L.ptr(ws), L.stream_ptr(stream)), "fc_loss_dense")
    return loss, crop, dl


def uniform_grid_device(seed, t, channel, row0, col0, height, width, stream=None) -> torch.Tensor:
    L.require_cuda()
    if height < 0 or width < 0:
        raise ValueError("negative window")
    out = torch.empty((max(height, 0), max(width, 0)), dtype=torch.float64, device="cuda")
    L.check(L.lib().fc_uniform_grid(int(seed) & (2**64 - 1), int(t), int(channel), int(row0),
                                    int(col0), int(height), int(width), L.ptr(out),
                                    L.stream_ptr(stream)), "fc_uniform_grid")
    return out


def build_fields_device(land: DeviceLandscape, params8, with_gradients=False, stream=None):
    L.require_cuda()
    h, w = land.shape
    g = L.grid(h, w, 1)
    p = torch.tensor(params8, dtype=torch.float64, device=land.env.device)
    out = torch.empty(((5 if with_gradients else 1) * 8, h, w), dtype=torch.float64,
                      device=land.env.device)
    lst = land.struct()
    L.check(L.lib().fc_build_fields(C.byref(g), C.byref(lst), L.ptr(p), L.ptr(out),
                                    1 if with_gradients else 0, L.stream_ptr(stream)),
            "fc_build_fields")
    return out


class CapturedSequence:
    """A CUDA graph of a device-only call sequence (e.g. one calibration
    iteration: reset + K-step windows + fused loss/gradient + AdamW).  Params,
    seeds and the Adam step live in device memory, so replays see updates."""

    def __init__(self, fn, warmup: int = 1):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            fn()

    def replay(self):
        self.graph.replay()
