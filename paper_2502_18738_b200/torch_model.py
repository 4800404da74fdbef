"""Torch model object with the paper's Algorithm 1 names.

    model = FireModel(landscape, init)            # a, c1, c2, p_h, p_continue, c
    model.reset(); seed = model.seed
    for step in ...: model.compute(attach=check_if_attach(step, n, rings))
    (or model.step(attach=...) per step, or model.run(n, rings=rings) fused)
    loss = criterion(model.accumulator, target); loss.backward()
    optimizer.step(); optimizer.zero_grad()
    with torch.no_grad(): model.a.clamp_(0, 1); ...; model.reset(seed=seed)

``model.accumulator`` is produced by a custom autograd.Function whose
backward is the device contraction sum_j dL/dacc_j * J_j (the straight-
through gradient of pyrocell/tape.py:118-148); p_continue receives zero
gradient exactly as in the reference.
"""
from __future__ import annotations

import os
from typing import Optional

import numpy as np
import torch
from torch import nn

from .device import DEFAULT_NORM_C, DeviceLandscape, FireBatch, loss_dense


class _Accumulator(torch.autograd.Function):
    @staticmethod
    def forward(ctx, c1, c2, a, p_h, p_continue, model):
        ctx.model = model
        ctx.dtypes = (c1.dtype, c2.dtype, a.dtype, p_h.dtype, p_continue.dtype)
        return model._batch.acc[0].clone()

    @staticmethod
    def backward(ctx, grad_acc):
        g = ctx.model._batch.contract(grad_acc.detach().unsqueeze(0))[0]
        dts = ctx.dtypes
        return (g[0].to(dts[0]), g[1].to(dts[1]), g[2].to(dts[2]), g[3].to(dts[3]),
                torch.zeros((), dtype=dts[4], device=g.device), None)


class _CombinedLoss(torch.autograd.Function):
    @staticmethod
    def forward(ctx, acc, target):
        loss, _, dl = loss_dense(acc.detach(), target)
        ctx.save_for_backward(dl)
        ctx.acc_dtype = acc.dtype
        return loss[0].to(acc.dtype)

    @staticmethod
    def backward(ctx, gout):
        (dl,) = ctx.saved_tensors
        return (dl * gout).to(ctx.acc_dtype), None


def combined_loss_torch(acc: torch.Tensor, target) -> torch.Tensor:
    """Differentiable combined_loss (losses.py:44-86) on the device kernel."""
    t = target if torch.is_tensor(target) else torch.as_tensor(np.asarray(target, dtype=bool))
    return _CombinedLoss.apply(acc, t.to(acc.device))


class FireModel(nn.Module):
    """Wildfire CA with trainable (a, c1, c2, p_h, p_continue) and constant c."""

    def __init__(self, landscape: DeviceLandscape, init, *, a=0.078, c1=0.045, c2=0.131,
                 p_h=0.58, p_continue=0.5, c=DEFAULT_NORM_C, max_steps: int = 4096,
                 rng: str = "splitmix", seed: Optional[int] = None):
        super().__init__()
        dev = landscape.env.device
        f64 = lambda v: nn.Parameter(torch.tensor(float(v), dtype=torch.float64, device=dev))
        self.a, self.c_1, self.c_2, self.p_h, self.p_continue = f64(a), f64(c1), f64(c2), \
            f64(p_h), f64(p_continue)
        self.register_buffer("c", torch.tensor(float(c), dtype=torch.float64, device=dev))
        self._base = landscape
        self._land = landscape
        self._init = init
        self._rng = rng
        self._batch = FireBatch(landscape.shape, 1, max_steps=max_steps, with_jacobian=True,
                                device=dev)
        self.seed = 0
        self.reset(seed)

    # Algorithm 1 aliases
    @property
    def c1(self):
        return self.c_1

    @property
    def c2(self):
        return self.c_2

    def reset(self, seed: Optional[int] = None):
        """Initial state; a fresh random seed unless one is given."""
        if seed is None:
            seed = int.from_bytes(os.urandom(8), "little")
        self.seed = int(seed)
        self._batch.set_seeds([self.seed])
        self._batch.reset(self._init)
        self._land = self._base

    @property
    def wind(self):
        return self._land.env64[..., 1], self._land.env64[..., 2]

    @wind.setter
    def wind(self, value):
        speed, direction = value
        if getattr(self, "_wind_src", None) is not value:
            self._land = self._base.with_wind(speed, direction)
            self._wind_src = value

    def _sync_params(self):
        with torch.no_grad():
            row = torch.stack([self.c_1, self.c_2, self.a, self.p_h, self.p_continue, self.c])
            self._batch.params[0, :6].copy_(row)

    def compute(self, attach: bool = False, steps: int = 1):
        """Advance `steps` steps; attached steps join the gradient."""
        self._sync_params()
        att = attach if isinstance(attach, (list, tuple, np.ndarray)) else [attach] * steps
        self._batch.run(self._land, steps, attach=att, rng=self._rng)

    def step(self, attach: bool = False):
        """One CA step (Algorithm 1's inner loop body)."""
        self.compute(attach=attach, steps=1)

    def run(self, steps: int, attach=False, rings=None):
        """Advance `steps` steps in fused launches.  attach: one flag for every
        step, or a per-step sequence; rings (StepRings): attach the steps of
        attachment_plan(self.t + steps, rings) -- check_if_attach over the
        whole re-simulation, as in Algorithm 1."""
        if steps < 0:
            raise ValueError("steps must be >= 0")
        if rings is not None:
            from .tape import attachment_plan
            total = self.t + steps
            plan = set(attachment_plan(total, rings))
            attach = [s in plan for s in range(self.t + 1, total + 1)]
        self.compute(attach=attach, steps=steps)

    @property
    def t(self) -> int:
        return self._batch.t

    @property
    def accumulator(self) -> torch.Tensor:
        return _Accumulator.apply(self.c_1, self.c_2, self.a, self.p_h, self.p_continue, self)

    def state(self):
        b, d = self._batch.unpack()
        return b[0].bool(), d[0].bool()

    def clamp_(self):
        with torch.no_grad():
            self.a.clamp_(0.0, 1.0)
            self.c_1.clamp_(0.0, 1.0)
            self.c_2.clamp_(0.0, 1.0)
            self.p_h.clamp_(0.2, 1.0)
