"""Ensemble forward runs from host buffers (the public call behind bench e2e).

``EnsembleRunner`` keeps device buffers and pinned host staging between calls:
each call uploads one landscape (fp32 rasters) and the initial mask, runs M
members for `steps` steps on the device (libfirecell fc_run) and copies the
final states, accumulators and per-step counts back to host memory.
"""
from __future__ import annotations

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


class EnsembleRunner:
    def __init__(self, shape, members: int, steps: int, *, cell_side: float = 30.0,
                 rng: str = "splitmix", device=None):
        self.h, self.w = shape
        self.m, self.steps, self.rng = int(members), int(steps), rng
        self.cell_side = cell_side
        self.batch = FireBatch(shape, members, max_steps=max(steps, 1), device=device)
        dev = self.batch.device
        self.dev = dev
        self.env_dev = torch.empty((5, self.h, self.w), dtype=torch.float32, device=dev)
        self.init_dev = torch.empty((self.h, self.w), dtype=torch.uint8, device=dev)
        self.out_b = _pinned((self.m, self.h, self.w), torch.uint8)
        self.out_d = _pinned((self.m, self.h, self.w), torch.uint8)
        self.out_acc = _pinned((self.m, self.h, self.w), torch.float32)
        self.out_cnt = _pinned((self.m, max(steps, 1), 4), torch.int32)
        self.out_init = _pinned((self.m,), torch.int64)
        self.in_params = _pinned((self.m, 8), torch.float64)
        self.in_seeds = _pinned((self.m,), torch.int64)
        self.copy_stream = torch.cuda.Stream(device=dev)
        self._graph = None  # CUDA graph of the device part (landscape, reset, run, unpack)
        self.h2d_bytes = self.env_dev.numel() * 4 + self.init_dev.numel()
        self.d2h_bytes = (self.out_b.numel() * 2 + self.out_acc.numel() * 4
                          + self.m * self.steps * 4 * 4)

    def __call__(self, env_host: torch.Tensor, init_host: torch.Tensor, params: Sequence,
                 seeds: Sequence[int], norm_c: float = DEFAULT_NORM_C,
                 sync: bool = True) -> EnsembleResult:
        """env_host: (5, H, W) fp32 (elevation, speed, direction, canopy,
        density), ideally pinned; init_host: (H, W) uint8/bool;
        params: per-member (c1, c2, a, p_h, p_continue)."""
        from .device import _u64_to_i64
        st = torch.cuda.current_stream(self.dev)
        st.wait_stream(self.copy_stream)  # the previous call's accumulator copy is done
        self.env_dev.copy_(env_host, non_blocking=True)
        self.init_dev.copy_(init_host, non_blocking=True)
        self.in_params.numpy()[:] = np.array([pack_params(*p, norm_c) for p in params],
                                             dtype=np.float64).reshape(self.m, -1)
        sd = [_u64_to_i64(v) for v in np.atleast_1d(np.asarray(seeds, dtype=object))]
        self.in_seeds.numpy()[:] = sd * self.m if len(sd) == 1 else sd
        self.batch.params.copy_(self.in_params, non_blocking=True)
        self.batch.seeds.copy_(self.in_seeds, non_blocking=True)
        # device part as one CUDA graph (built on the first call): the
        # landscape preparation, reset, the window launches and the unpack
        if self._graph is None:
            from .device import CapturedSequence
            self._graph = CapturedSequence(self._device_part)
        self._graph.replay()
        # the accumulator leaves on a side stream while the states leave here
        done = torch.cuda.Event()
        done.record(st)
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(done)
            self.out_acc.copy_(self.batch.acc, non_blocking=True)
        b, d = self._bu, self._bd
        self.out_b.copy_(b, non_blocking=True)
        self.out_d.copy_(d, non_blocking=True)
        self.out_cnt.copy_(self.batch.counters[:, : max(self.steps, 1)], non_blocking=True)
        self.out_init.copy_(self.batch._init_burning_dev, non_blocking=True)
        self.batch.acc.record_stream(self.copy_stream)
        if sync:
            st.synchronize()
            self.copy_stream.synchronize()
        cnt = self.out_cnt.numpy()[:, : self.steps].astype(np.int64)
        burning = self.out_init.numpy()[:, None] + np.cumsum(cnt[:, :, 0] - cnt[:, :, 1], axis=1)
        burned = np.cumsum(cnt[:, :, 1], axis=1)
        return EnsembleResult(self.out_b.numpy(), self.out_d.numpy(), self.out_acc.numpy(),
                              np.stack([burning, burned], axis=-1))

    def _device_part(self):
        e = self.env_dev
        land = DeviceLandscape.from_elevation(e[0], e[1], e[2], e[3], e[4],
                                              cell_side=self.cell_side, device=self.dev)
        self._land = land  # keeps the graph's landscape buffers referenced
        self.batch.reset(self.init_dev)
        self.batch.run(land, self.steps, rng=self.rng)
        self._bu, self._bd = self.batch.unpack()


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
                 lr: float = 1e-2, weight_decay: float = 0.0, window: int = 8, device=None):
        from .parallel import allreduce_sum_  # noqa: F401  (import check)
        self.land, self.lr, self.wd, self.window = land, lr, weight_decay, window
        self.steps = int(steps if steps is not None else max(obs_steps))
        self.obs = [int(s) for s in obs_steps]
        self.batch = FireBatch(land.shape, len(members), max_steps=self.steps,
                               with_jacobian=True, device=device)
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

    def step(self):
        """One iteration; returns the (members, 2 + 2S) loss rows (device)."""
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
