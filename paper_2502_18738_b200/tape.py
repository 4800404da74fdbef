"""Attachment plan and the device-side gradient tape (API of pyrocell/tape.py).

The reference records, per attached step, (n, 8) caches of every newly
ignited cell and contracts them in backward_params (tape.py:118-148).  Here
the step kernel records each ignition's live-slot mask; fc_recompute64
turns masks into fp64 p_ignite and J_j = dp_j/d(c1, c2, a, p_h) with the
reference's operation order, and the backward is one contraction
sum_j dL/dacc_j * J_j on the device (fc_contract_steps).  The reference's
TapeBlocks are materialised from the same device record when read.
Straight-through semantics are unchanged: the realised trajectory is
constant (tape.py:1-7).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

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


@dataclass
class TapeBlock:
    """tape.py:49-87: one attached step's newly ignited cells, (n, 8) caches
    over the slot order (zero on dead slots), rows in row-major cell order.

    Blocks of a device run are materialised on demand from the run's
    live-slot masks and the fp64 fields of the step's landscape
    (fc_build_fields); p_ignite is the fp64 recomputation fc_recompute64
    stores in the run's accumulator, so recombine() reproduces it bit for
    bit, as in the reference."""

    t: int
    rows: np.ndarray
    cols: np.ndarray
    p_ignite: np.ndarray
    mask: np.ndarray
    fp: np.ndarray
    raw: np.ndarray
    rest: np.ndarray
    vw: np.ndarray
    cosm1: np.ndarray
    slope: np.ndarray
    veg1: np.ndarray
    den1: np.ndarray
    _src: Optional["RunBinding"] = field(default=None, repr=False, compare=False)

    def __len__(self) -> int:
        return int(self.rows.size)

    def recombine(self) -> np.ndarray:
        """tape.py:77-87: 1 - prod over slots of (1 - fp), frozen slot order."""
        factors = np.where(self.mask, 1.0 - self.fp, 1.0)
        prod = np.ones(len(self), dtype=np.float64)
        for k in range(8):
            prod *= factors[:, k]
        return 1.0 - prod


class RunBinding:
    """The device record of one run's attached steps: the batch (t_ign,
    live-slot masks), the fp64 Jacobians of its ignitions (fc_recompute64)
    and the landscape of every step segment, from which TapeBlocks are
    materialised on demand."""

    def __init__(self, batch, jac64: torch.Tensor, acc64: torch.Tensor, segments,
                 attached_steps, entries_per_step: dict, norm_c: float, canopy, density,
                 site_is_target: bool):
        self.batch, self.jac64, self.acc64 = batch, jac64, acc64
        self.segments = segments          # [(t_lo, t_hi, DeviceLandscape, params8, wind speed)]
        self.steps = tuple(int(s) for s in attached_steps)  # 1-based, sorted
        self.entries = dict(entries_per_step)                # 1-based step -> ignitions
        self.norm_c = float(norm_c)
        self.canopy, self.density, self.site_is_target = canopy, density, site_is_target
        self._blocks: Optional[List[TapeBlock]] = None

    @property
    def num_entries(self) -> int:
        return int(sum(self.entries.get(s, 0) for s in self.steps))

    def blocks(self) -> List[TapeBlock]:
        if self._blocks is None:
            self._blocks = self._materialise()
        return self._blocks

    def _materialise(self) -> List[TapeBlock]:
        from .device import NEIGHBOR_POSITIONS, build_fields_device
        t_ign = self.batch.t_ign[0]
        live = self.batch.live[0]
        h, w = t_ign.shape
        out = []
        fields_cache = {}
        for s in self.steps:
            t = s - 1
            if not self.entries.get(s, 0):
                continue
            seg = next(g for g in self.segments if g[0] <= t < g[1])
            key = id(seg[2])
            if key not in fields_cache:
                fields_cache.clear()
                fields_cache[key] = build_fields_device(seg[2], seg[3], with_gradients=True)
            F = fields_cache[key]
            # t_ign counts from the batch's base; row-major, as np.nonzero (kernel.py:345-347)
            idx = torch.nonzero(t_ign == t - self.batch.t_base)
            rows, cols = idx[:, 0], idx[:, 1]
            n = rows.numel()
            bits = live[rows, cols].to(torch.int32)
            cache = {k: torch.zeros((n, 8), dtype=torch.float64, device=F.device)
                     for k in ("fp", "raw", "rest", "vw", "cosm1", "slope", "veg1", "den1")}
            mask = torch.zeros((n, 8), dtype=torch.bool, device=F.device)
            vw = torch.as_tensor(np.asarray(seg[4], dtype=np.float64), device=F.device)
            can = torch.as_tensor(np.asarray(self.canopy, dtype=np.float64), device=F.device)
            den = torch.as_tensor(np.asarray(self.density, dtype=np.float64), device=F.device)
            for k, (pr, pc) in enumerate(NEIGHBOR_POSITIONS):
                lv = ((bits >> k) & 1).bool()
                mask[:, k] = lv
                sr, sc = (rows + pr)[lv], (cols + pc)[lv]
                for name, plane in (("fp", 0), ("raw", 8), ("rest", 16), ("cosm1", 24),
                                    ("slope", 32)):
                    cache[name][lv, k] = F[plane + k][sr, sc]
                cache["vw"][lv, k] = vw[sr, sc]
                site_r, site_c = (rows[lv], cols[lv]) if self.site_is_target else (sr, sc)
                cache["veg1"][lv, k] = 1.0 + can[site_r, site_c]
                cache["den1"][lv, k] = 1.0 + den[site_r, site_c]
            host = {k: v.cpu().numpy() for k, v in cache.items()}
            out.append(TapeBlock(t=t, rows=rows.cpu().numpy(), cols=cols.cpu().numpy(),
                                 p_ignite=self.acc64[0][rows, cols].cpu().numpy(),
                                 mask=mask.cpu().numpy(), _src=self, **host))
        return out


class Tape:
    """tape.py:90-103: append-only record of attached steps.  Entries are
    device runs (RunBinding: fp64 Jacobians of every attached ignition, the
    blocks materialised when ``blocks`` is read) or explicit TapeBlocks."""

    def __init__(self, shape, blocks: Optional[Sequence[TapeBlock]] = None):
        self.shape = tuple(int(v) for v in shape)
        self._entries: list = list(blocks) if blocks is not None else []
        self.norm_c: Optional[float] = None

    def add_block(self, block: TapeBlock) -> None:
        self._entries.append(block)

    def bind(self, binding: RunBinding) -> None:
        self._entries.append(binding)
        self.norm_c = binding.norm_c

    @property
    def blocks(self) -> List[TapeBlock]:
        out: List[TapeBlock] = []
        for e in self._entries:
            out.extend(e.blocks() if isinstance(e, RunBinding) else [e])
        return out

    @property
    def num_entries(self) -> int:
        return int(sum(e.num_entries if isinstance(e, RunBinding) else len(e)
                       for e in self._entries))

    def __len__(self) -> int:
        return self.num_entries


def backward_params(tape: Tape, dl_dacc, norm_c: float) -> np.ndarray:
    """tape.py:118-148 -> (dc1, dc2, da, dp_h), in fp64 on the device: a
    run's attached steps contract dL/dacc with its fp64 Jacobians
    (fc_contract_steps, J from fc_recompute64); blocks taken from a run
    contract the same way over their steps; hand-made blocks use their own
    caches (the reference's leave-one-out chain)."""
    g = np.asarray(dl_dacc) if not torch.is_tensor(dl_dacc) else dl_dacc
    if tuple(g.shape) != tape.shape:
        raise ValueError(f"loss grid {tuple(g.shape)} != tape grid {tape.shape}")
    grad = np.zeros(4, dtype=np.float64)
    by_run: dict = {}
    loose: List[TapeBlock] = []
    for e in tape._entries:
        if isinstance(e, RunBinding):
            by_run.setdefault(id(e), (e, set()))[1].update(s - 1 for s in e.steps)
        elif e._src is not None:
            by_run.setdefault(id(e._src), (e._src, set()))[1].add(int(e.t))
        else:
            loose.append(e)
    for run, steps in by_run.values():
        if not steps:
            continue
        gt = torch.as_tensor(g, dtype=torch.float64).to(run.jac64.device) \
            if not torch.is_tensor(g) else g.to(run.jac64.device, torch.float64)
        out = run.batch.contract_steps(gt, run.jac64, sorted(steps))[0].cpu().numpy()
        # the chain carries the explicit factor c (tape.py:134-140)
        grad += out * (float(norm_c) / run.norm_c)
    if loose:
        grad += _blocks_backward(loose, g, norm_c)
    return grad


def _blocks_backward(blocks: Sequence[TapeBlock], g, norm_c: float) -> np.ndarray:
    """The reference chain (tape.py:106-148) over hand-made blocks, fp64 on
    the device."""
    from . import _lib as L
    L.require_cuda()
    dev = torch.device("cuda")
    gt = torch.as_tensor(np.asarray(g, dtype=np.float64) if not torch.is_tensor(g) else g,
                         dtype=torch.float64, device=dev)
    grad = torch.zeros(4, dtype=torch.float64, device=dev)
    for b in blocks:
        if len(b) == 0:
            continue
        T = lambda a: torch.as_tensor(np.asarray(a), device=dev)
        mask, fp = T(b.mask), T(b.fp).double()
        fac = torch.where(mask, 1.0 - fp, torch.ones_like(fp))
        pre = torch.cumprod(torch.cat([torch.ones_like(fac[:, :1]), fac[:, :-1]], 1), 1)
        suf = torch.flip(torch.cumprod(torch.cat([torch.ones_like(fac[:, :1]),
                                                  torch.flip(fac, [1])[:, :-1]], 1), 1), [1])
        gv = gt[T(b.rows).long(), T(b.cols).long()]
        chain = gv[:, None] * (pre * suf) * (norm_c * (1.0 - fp * fp)) * mask
        raw, vw = T(b.raw).double(), T(b.vw).double()
        grad[0] += torch.sum(chain * raw * vw)
        grad[1] += torch.sum(chain * raw * vw * T(b.cosm1).double())
        grad[2] += torch.sum(chain * raw * T(b.slope).double())
        grad[3] += torch.sum(chain * T(b.rest).double())
    return grad.cpu().numpy()
