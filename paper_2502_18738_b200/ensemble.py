"""Ensemble forward runs from host buffers (the public call behind bench e2e).

``EnsembleRunner`` keeps device buffers and pinned host staging between calls:
each call uploads one landscape (fp32 rasters) and the initial mask, runs M
members for `steps` steps on the device (libfirecell fc_run) and copies the
final states, accumulators and per-step counts back to host memory.

Calls can be pipelined: ``submit`` queues one call and returns a ticket
whose ``result()`` waits for that call's outputs.  The runner holds
``depth`` slots (device buffers, a captured CUDA graph of the device part,
pinned inputs and outputs each).  Three streams overlap: uploads of call
i+1, the kernels of call i, and the export of call i-1 -- fc_state_export
writes the result arrays in pinned host memory directly from the bit planes,
touching only tiles that are affected now or were written by the slot's
previous call (everywhere else the arrays already hold zeros), so the PCIe
traffic is the fire's footprint, not the grid.  A result's arrays are
read-only views of its slot's buffers, valid until ``depth`` further
submissions.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from .device import DEFAULT_NORM_C, DeviceLandscape, FireBatch, pack_params


@dataclass
class EnsembleResult:
    burning: np.ndarray   # (M, H, W) uint8
    burned: np.ndarray    # (M, H, W) uint8
    accumulator: np.ndarray  # (M, H, W) fp32
    series: np.ndarray    # (M, steps, 2) int64 (burning, burned after each step)


def _pinned(shape, dtype):
    return torch.empty(shape, dtype=dtype, pin_memory=True)


class _Slot:
    """One pipeline stage: device state + graph + pinned staging.  The
    result arrays are pinned host memory the export kernel writes directly
    (zero-initialised once; per-tile ``written`` flags keep them exact)."""

    def __init__(self, runner: "EnsembleRunner", device):
        from . import _lib as L
        r = runner
        self.batch = FireBatch((r.h, r.w), r.m, max_steps=max(r.steps, 1), member0=r.member0,
                               device=device)
        dev = self.batch.device
        g = self.batch.grid
        self.env_dev = torch.empty((5, r.h, r.w), dtype=torch.float32, device=dev)
        self.init_dev = torch.empty((r.h, r.w), dtype=torch.uint8, device=dev)
        # the kernel-layout landscape of the slot, rebuilt in place each call
        # (fc_landscape_build_ctas on the upload stream)
        env = torch.zeros((r.h, r.w, 4), dtype=torch.float32, device=dev)
        env64 = torch.zeros((r.h, r.w, 5), dtype=torch.float64, device=dev)
        slope4 = torch.zeros((r.h, r.w, 4), dtype=torch.float32, device=dev)
        dir32 = torch.zeros((r.h, r.w, 2), dtype=torch.float32, device=dev)
        self.land = DeviceLandscape(env, env64, cell_side=r.cell_side, slope4=slope4, dir32=dir32)
        self.out_b = torch.zeros((r.m, r.h, r.w), dtype=torch.uint8, pin_memory=True)
        self.out_d = torch.zeros((r.m, r.h, r.w), dtype=torch.uint8, pin_memory=True)
        self.out_acc = torch.zeros((r.m, r.h, r.w), dtype=torch.float32, pin_memory=True)
        self.written = torch.zeros((r.m, g.tiles_y, g.tiles_x), dtype=torch.uint8, device=dev)
        self.out_ptrs = [L.device_ptr(t) for t in (self.out_b, self.out_d, self.out_acc)]
        self.out_cnt = _pinned((r.m, max(r.steps, 1), 4), torch.int32)
        self.out_init = _pinned((r.m,), torch.int64)
        self.in_params = _pinned((r.m, 8), torch.float64)
        self.in_seeds = _pinned((r.m,), torch.int64)
        self.uploaded = None   # event: this slot's pinned inputs have been read
        self.computed = None   # event: this slot's device part has run
        self.copied = None     # event: this slot's outputs are in host memory
        self.graph = None
        self.runner = r

    def build_landscape(self, stream, max_ctas: int):
        """fc_landscape_build_ctas from the uploaded rasters into the slot's
        landscape buffers (bit-identical to DeviceLandscape.from_elevation)."""
        from . import _lib as L
        e, land = self.env_dev, self.land
        with torch.cuda.device(self.batch.device):  # the launch goes to this device
            L.check(L.lib().fc_landscape_build_ctas(
                self.runner.h, self.runner.w, *[L.ptr(e[i]) for i in range(5)], 0,
                float(self.runner.cell_side), 1, L.ptr(land.env), L.ptr(land.slope4),
                L.ptr(land.env64), L.ptr(land.dir32), int(max_ctas), L.stream_ptr(stream)),
                "fc_landscape_build_ctas")

    def device_part(self):
        self.batch.reset(self.init_dev)
        self.batch.run(self.land, self.runner.steps, rng=self.runner.rng)

    def export(self, stream):
        """fc_state_export into the pinned result arrays + the counters."""
        import ctypes as C
        from . import _lib as L
        b = self.batch
        st = b.struct()
        with torch.cuda.device(b.device):
            L.check(L.lib().fc_state_export(C.byref(b.grid), C.byref(st), b.q, *self.out_ptrs,
                                            L.ptr(self.written), L.stream_ptr(stream)),
                    "fc_state_export")
        self.out_cnt.copy_(b.counters[:, : max(self.runner.steps, 1)], non_blocking=True)
        self.out_init.copy_(b._init_burning_dev, non_blocking=True)


class EnsembleTicket:
    """A submitted call; result() blocks until its outputs are on the host."""

    def __init__(self, slot: _Slot, steps: int):
        self.slot, self.steps, self.event = slot, steps, slot.copied
        self.inputs_consumed = slot.uploaded  # the H2D copies of this call's inputs are done

    def done(self) -> bool:
        return self.event.query()

    def wait_inputs(self) -> None:
        """Block until this call has read the caller's host input buffers
        (env_host, init_host): only then may the caller refill them.  submit()
        returns before the asynchronous copies run (that is what lets the
        upload overlap the previous call's kernels)."""
        self.inputs_consumed.synchronize()

    def result(self) -> EnsembleResult:
        self.event.synchronize()
        s = self.slot
        cnt = s.out_cnt.numpy()[:, : self.steps].astype(np.int64)
        burning = s.out_init.numpy()[:, None] + np.cumsum(cnt[:, :, 0] - cnt[:, :, 1], axis=1)
        burned = np.cumsum(cnt[:, :, 1], axis=1)
        arrays = [s.out_b.numpy(), s.out_d.numpy(), s.out_acc.numpy()]
        for a in arrays:  # the slot's buffers are reused: callers copy to keep or modify
            a.flags.writeable = False
        return EnsembleResult(*arrays, np.stack([burning, burned], axis=-1))

    def exported_tiles(self) -> int:
        """Tiles the export wrote (after result(); syncs)."""
        return int(self.slot.written.sum())


class EnsembleRunner:
    def __init__(self, shape, members: int, steps: int, *, cell_side: float = 30.0,
                 rng: str = "splitmix", depth: int = 2, member0: int = 0, device=None):
        """member0: global index of this runner's first member when an
        ensemble is sharded over ranks (keys the Philox draws)."""
        self.h, self.w = shape
        self.member0 = int(member0)
        self.m, self.steps, self.rng = int(members), int(steps), rng
        self.cell_side = cell_side
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.slots = [_Slot(self, device) for _ in range(depth)]
        self.dev = self.slots[0].batch.device
        self.batch = self.slots[0].batch
        # the kernels run on a high-priority stream; the export's short CTAs
        # (low priority) fill SMs the step kernel leaves idle
        self.compute_stream = torch.cuda.Stream(device=self.dev, priority=-5)
        self.upload_stream = torch.cuda.Stream(device=self.dev, priority=0)
        # CTAs of the landscape build (0 = the full grid): its fp64 slope
        # arithmetic needs the whole GPU -- on 4 / 8 / 16 / 32 CTAs a c1 call
        # took 13.3 / 8.0 / 5.8 / 4.9 ms against 3.6 ms with the full grid
        self.landscape_ctas = int(os.environ.get("FC_LANDSCAPE_CTAS", 0))
        self.copy_stream = torch.cuda.Stream(device=self.dev, priority=0)
        self._next = 0
        s0 = self.slots[0]
        self.h2d_bytes = s0.env_dev.numel() * 4 + s0.init_dev.numel() + self.m * (8 + 1) * 8
        # full-grid equivalent; the export writes only affected tiles
        self.d2h_bytes_dense = (s0.out_b.numel() * 2 + s0.out_acc.numel() * 4
                                + self.m * self.steps * 4 * 4)

    def d2h_bytes(self, ticket: EnsembleTicket) -> int:
        """Bytes one call moved device -> host (after result(); syncs): the
        export writes whole 128-column spans (4 tiles) that hold a written
        tile, 1 + 1 + 4 B per cell, plus the per-step counters.  Counted from
        the slot's written flags, i.e. exact when consecutive calls affect the
        same tiles (the bench repeats one workload)."""
        g = ticket.slot.batch.grid
        w = ticket.slot.written.to(torch.bool).cpu().numpy()          # (M, TY, TX)
        span = 4
        nsp = (g.tiles_x + span - 1) // span
        pad = np.zeros((w.shape[0], w.shape[1], nsp * span), dtype=bool)
        pad[:, :, : g.tiles_x] = w
        dirty = pad.reshape(w.shape[0], w.shape[1], nsp, span).any(-1)  # (M, TY, nsp)
        rows = np.minimum(32, self.h - 32 * np.arange(g.tiles_y))[:, None]
        cols = np.minimum(128, self.w - 128 * np.arange(nsp))[None, :]
        cells = int((dirty * (rows * cols)[None]).sum())
        return cells * 6 + self.m * (self.steps * 16 + 8)

    def submit(self, env_host: torch.Tensor, init_host: torch.Tensor, params: Sequence,
               seeds: Sequence[int], norm_c: float = DEFAULT_NORM_C) -> EnsembleTicket:
        """Queue one call.  env_host: (5, H, W) fp32 (elevation, speed,
        direction, canopy, density), ideally pinned; init_host: (H, W)
        uint8/bool; params: per-member (c1, c2, a, p_h, p_continue).
        The host inputs are read asynchronously: a caller that refills the
        same buffers for the next call must first wait for
        ``ticket.wait_inputs()`` (or ``result()``).

        Streams: uploads and the landscape build on upload_stream,
        overlapping the previous call's kernels; the device
        part (one CUDA graph: reset and run) on the high-priority
        compute_stream, after the work the caller's current stream holds;
        the export (kernel writing pinned host memory) on copy_stream."""
        from .device import CapturedSequence, _u64_to_i64
        slot = self.slots[self._next]
        self._next = (self._next + 1) % len(self.slots)
        caller = torch.cuda.current_stream(self.dev)
        st, us, cs = self.compute_stream, self.upload_stream, self.copy_stream
        st.wait_stream(caller)                 # work the caller queued before this call
        if slot.uploaded is not None:
            slot.uploaded.synchronize()        # its pinned inputs are free to refill
        slot.in_params.numpy()[:] = np.array([pack_params(*p, norm_c) for p in params],
                                             dtype=np.float64).reshape(self.m, -1)
        sd = [_u64_to_i64(v) for v in np.atleast_1d(np.asarray(seeds, dtype=object))]
        slot.in_seeds.numpy()[:] = sd * self.m if len(sd) == 1 else sd
        if slot.graph is None:
            # first use: capture the device part (landscape preparation,
            # reset, the window launches) as one graph on the current stream
            slot.env_dev.copy_(env_host)
            slot.init_dev.copy_(init_host)
            slot.batch.params.copy_(slot.in_params)
            slot.batch.seeds.copy_(slot.in_seeds)
            slot.build_landscape(caller, 0)
            with torch.cuda.stream(st):
                st.wait_stream(caller)
                slot.graph = CapturedSequence(slot.device_part)
        with torch.cuda.stream(us):
            # inputs the caller produced on its stream (device-side writes to
            # pinned buffers, or a preceding call's results) come first
            us.wait_stream(caller)
            if slot.computed is not None:
                us.wait_event(slot.computed)   # its previous run has read the inputs
            slot.env_dev.copy_(env_host, non_blocking=True)
            slot.init_dev.copy_(init_host, non_blocking=True)
            slot.batch.params.copy_(slot.in_params, non_blocking=True)
            slot.batch.seeds.copy_(slot.in_seeds, non_blocking=True)
            # the landscape of this call, built next to the previous call's
            # step kernels
            slot.build_landscape(us, self.landscape_ctas)
            slot.uploaded = torch.cuda.Event()
            slot.uploaded.record(us)
        st.wait_event(slot.uploaded)
        if slot.copied is not None:
            st.wait_event(slot.copied)         # its previous export has read the state
        with torch.cuda.stream(st):
            slot.graph.replay()
        slot.computed = torch.cuda.Event()
        slot.computed.record(st)
        with torch.cuda.stream(cs):
            cs.wait_event(slot.computed)
            slot.export(cs)
            slot.copied = torch.cuda.Event()
            slot.copied.record(cs)
        return EnsembleTicket(slot, self.steps)

    def __call__(self, env_host: torch.Tensor, init_host: torch.Tensor, params: Sequence,
                 seeds: Sequence[int], norm_c: float = DEFAULT_NORM_C) -> EnsembleResult:
        """One synchronous call (submit + result)."""
        return self.submit(env_host, init_host, params, seeds, norm_c).result()


def _graph_safe_collectives() -> bool:
    """Whether the iteration is captured as a CUDA graph: one process only.
    With several ranks the all-reduce stays eager -- a capture that failed on
    one rank and not on another would leave the ranks' collectives
    mismatched (the graph saves ~1 % of a c4 iteration)."""
    import torch.distributed as dist
    return not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1


class EnsembleCalibrator:
    """Ensemble fwd+bwd calibration (BASELINE config 4) on this rank's
    members: every iteration re-simulates all members from the initial state
    with every step attached, sums the per-member loss gradients (fused
    loss/contraction kernel), all-reduces the 4 fp64 gradients over ranks
    (NCCL) and applies one AdamW + clamp step to the shared parameters, which
    all ranks therefore keep identical."""

    def __init__(self, land: DeviceLandscape, init, targets: torch.Tensor,
                 obs_steps: Sequence[int], members: Sequence[int], params, *,
                 steps: Optional[int] = None, wind_schedule: Optional[torch.Tensor] = None,
                 lr: float = 1e-2, weight_decay: float = 0.0, window: Optional[int] = None,
                 device=None, graph: bool = True):
        from .parallel import allreduce_sum_  # noqa: F401  (import check)
        self.land, self.lr, self.wd, self.window = land, lr, weight_decay, window
        self.steps = int(steps if steps is not None else max(obs_steps))
        self.obs = [int(s) for s in obs_steps]
        members = list(members)
        if members != list(range(members[0], members[0] + len(members))):
            raise ValueError("members must be a contiguous block (parallel.shard_members)")
        self.batch = FireBatch(land.shape, len(members), max_steps=self.steps,
                               with_jacobian=True, member0=members[0], device=device)
        dev = self.batch.device
        self.init = init if torch.is_tensor(init) else torch.as_tensor(
            np.asarray(init, dtype=bool).astype(np.uint8), device=dev)
        self.targets = targets.to(dev)
        self.wind = wind_schedule
        self.batch.set_seeds(list(members))
        self.shared = torch.as_tensor(np.asarray(pack_params(*params), dtype=np.float64),
                                      device=dev).reshape(1, -1).clone()
        self.adam = torch.zeros((1, 8), dtype=torch.float64, device=dev)
        self.adam_step = torch.zeros((1,), dtype=torch.int32, device=dev)
        self.attach = [True] * self.steps
        self.last_loss = None
        # iterations after the first replay one CUDA graph of the whole
        # iteration (reset, the run, loss/gradient, all-reduce, AdamW): the
        # host's per-launch work leaves the GPU's critical path
        self.use_graph, self._graph = bool(graph) and _graph_safe_collectives(), None

    def step(self):
        """One iteration; returns the (members, 2 + 2S) loss rows (device;
        with graph=True the same tensor every iteration, rewritten in place)."""
        if not self.use_graph:
            return self._iteration()
        if self._graph is None:
            from .device import CapturedSequence
            loss = self._iteration()
            try:
                # the capture records without executing (no second update)
                self._graph = CapturedSequence(self._iteration, warmup=0)
            except Exception:  # e.g. a collective that cannot be captured: stay eager
                torch.cuda.synchronize(self.batch.device)
                self.use_graph, self._graph = False, None
            self.last_loss = loss if self._graph is None else self.last_loss
            return loss
        self._graph.replay()
        return self.last_loss

    def _iteration(self):
        from . import _lib as L
        from .parallel import allreduce_sum_
        b = self.batch
        b.params.copy_(self.shared.expand_as(b.params))
        b.reset(self.init)
        b.run(self.land, self.steps, attach=self.attach, wind_schedule=self.wind,
              window=self.window)
        loss, _, grad, _ = b.loss_grad(self.targets, self.obs)
        g = grad.sum(0, keepdim=True)
        allreduce_sum_(g)
        L.check(L.lib().fc_adamw(L.ptr(g), L.ptr(self.shared), L.ptr(self.adam), 1, 0,
                                 L.ptr(self.adam_step), self.lr, self.wd, 0.9, 0.999, 1e-8, 1,
                                 None, L.stream_ptr()), "fc_adamw")
        self.last_loss = loss
        return loss

    @property
    def params(self) -> np.ndarray:
        return self.shared[0, :5].cpu().numpy()
