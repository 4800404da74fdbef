"""Attachment plan and the device-side gradient tape (API of pyrocell/tape.py).

The reference records, per attached step, (n, 8) caches of every newly
ignited cell and contracts them in backward_params (tape.py:118-148).  Here
the forward kernel writes each attached ignition's Jacobian
J_j = dp_j/d(c1, c2, a, p_h) once (fp32, HBM), and the backward is a single
contraction sum_j dL/dacc_j * J_j on the device.  Straight-through semantics
are unchanged: the realised trajectory is constant (tape.py:1-7).
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np
import torch

from .model import StepRings


def attachment_plan(total_steps: int, rings: StepRings) -> Tuple[int, ...]:
    """tape.py:19-39: first r_first, last r_last and r_between evenly spaced
    interior steps (NumPy rounding: half to even)."""
    if total_steps < 0:
        raise ValueError("total_steps must be >= 0")
    steps = set(range(1, min(rings.r_first, total_steps) + 1))
    steps |= set(range(max(total_steps - rings.r_last, 0) + 1, total_steps + 1))
    lo, hi = rings.r_first + 1, total_steps - rings.r_last + 1
    if rings.r_between > 0 and hi > lo:
        inner = np.linspace(lo, hi, rings.r_between + 2)[1:-1]
        steps |= {int(s) for s in np.round(inner).astype(int) if 1 <= s <= total_steps}
    return tuple(sorted(steps))


def check_if_attach(step: int, total_steps: int, rings: StepRings) -> bool:
    """tape.py:42-46."""
    if not 1 <= step <= total_steps:
        raise ValueError(f"step {step} outside 1..{total_steps}")
    return step in attachment_plan(total_steps, rings)


class Tape:
    """Gradient record of one run: a view of the run's device Jacobians.

    num_entries counts ignitions on attached steps (one logical tape entry
    per ignited cell, as in tape.py:49-103)."""

    def __init__(self, shape):
        self.shape = tuple(int(v) for v in shape)
        self.num_entries = 0
        self.jac: Optional[torch.Tensor] = None   # (H, W, 4) fp32 device
        self.norm_c: Optional[float] = None
        self.attached_steps: Tuple[int, ...] = ()
        self._batch = None

    def __len__(self) -> int:
        return self.num_entries

    def bind(self, batch, attached_steps, entries: int, norm_c: float):
        self._batch = batch
        self.jac = batch.jac[0]
        self.attached_steps = tuple(attached_steps)
        self.num_entries += int(entries)
        self.norm_c = float(norm_c)

    def accumulate(self, jac: torch.Tensor, step: int, entries: int, norm_c: float):
        """Add one step's Jacobians (step_forward with attach=True)."""
        if self.jac is None:
            self.jac = torch.zeros_like(jac)
        self.jac += jac
        self.attached_steps = self.attached_steps + (int(step),)
        self.num_entries += int(entries)
        self.norm_c = float(norm_c)


def backward_params(tape: Tape, dl_dacc, norm_c: float) -> np.ndarray:
    """tape.py:118-148 -> (dc1, dc2, da, dp_h)."""
    g = np.asarray(dl_dacc) if not torch.is_tensor(dl_dacc) else dl_dacc
    if tuple(g.shape) != tape.shape:
        raise ValueError(f"loss grid {tuple(g.shape)} != tape grid {tape.shape}")
    if tape.jac is None or tape.num_entries == 0:
        return np.zeros(4, dtype=np.float64)
    from .device import FireBatch  # noqa: F401  (lib loaded by the batch)
    gt = torch.as_tensor(g, dtype=torch.float64).to(tape.jac.device) if not torch.is_tensor(g) \
        else g.to(tape.jac.device)
    # a bound run's plane is valid where its cells ignited (t_ign gates it)
    tig = tape._batch.t_ign[0] if tape._batch is not None else None
    out = _contract(tape.jac, gt, tig)
    # chain_k carries the explicit factor c (tape.py:134-140): rescale when
    # the caller's constant differs from the forward's
    scale = float(norm_c) / tape.norm_c if tape.norm_c else 1.0
    return out * scale


def _contract(jac: torch.Tensor, g: torch.Tensor, t_ign: Optional[torch.Tensor] = None) -> np.ndarray:
    import ctypes as C
    from . import _lib as L
    h, w = jac.shape[:2]
    grid = L.grid(h, w, 1)
    st = L.FcState()
    st.jac = L.ptr(jac)
    st.acc = 0
    st.t_ign = 0 if t_ign is None else L.ptr(t_ign)
    gg = g.contiguous()
    ws = torch.empty((max(L.lib().fc_loss_workspace_bytes(C.byref(grid), 1), 4096),),
                     dtype=torch.uint8, device=jac.device)
    out = torch.empty((1, 4), dtype=torch.float64, device=jac.device)
    L.check(L.lib().fc_contract(C.byref(grid), C.byref(st), L.ptr(gg),
                                1 if gg.dtype == torch.float32 else 0, L.ptr(out), L.ptr(ws),
                                L.stream_ptr()), "fc_contract")
    return out[0].cpu().numpy()
